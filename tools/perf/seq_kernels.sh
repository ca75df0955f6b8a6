# per-kernel warm durations of the cfg4 iteration for each library variant (ncu launch list)
for v in "$@"; do
  if [ "$v" = main ]; then L=""; else L="MDHP_LIB=tools/ab/$v/libmdhp.so"; fi
  env $L ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_seq --csv \
    --log-file gpurun_out/seqk_${v}_${CHUNK:-256}.csv python bench.py --config cfg4 --steps 1 --warmup 3 --iters 10 --chunk ${CHUNK:-256} --no-cpu --no-e2e > /dev/null 2>&1
done
