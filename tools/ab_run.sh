#!/bin/bash
# A/B: run the bench probe once per variant library (on the GPU box).  Usage: tools/ab_run.sh "args" v1 v2 ...
args=$1; shift
for v in "$@"; do
  r=$(MDHP_LIB=/root/repo/tools/ab/$v/libmdhp.so python bench.py $args 2>&1 | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[2]); print(sys.argv[1], '%.4g' % d['value'], 'fit_ms %.1f' % d['roofline']['fit_ms_avg'], 'sm_mhz', d['clocks']['sm_mhz'])" "$v" "$r" 2>/dev/null || echo "$v FAILED: $r" | cut -c1-300
done
