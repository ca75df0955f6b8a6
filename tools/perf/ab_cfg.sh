# A/B: bench one config with the in-tree library and a tools/ab/<variant> library.
# usage: tools/perf/ab_cfg.sh <variant> <config> [extra bench args]
v=$1; cfg=$2; shift 2
for lib in main $v; do
  if [ "$lib" = main ]; then L=""; else L="MDHP_LIB=tools/ab/$lib/libmdhp.so"; fi
  r=$(env $L python bench.py --config $cfg --no-cpu --no-e2e --steps 2 --warmup 3 "$@" 2>&1 | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[3]); print(sys.argv[1], sys.argv[2], '%.4g' % d['value'])" $cfg $lib "$r" 2>/dev/null || echo "$cfg $lib FAIL ${r:0:200}"
done
