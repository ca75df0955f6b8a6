#!/bin/bash
# ncu --set full of one warm launch of a cfg4 phase kernel (default k_seq_eval) of the cfg4 fit
# (bench.py --config cfg4), exported as raw + SASS-source CSVs into gpurun_out/<kernel>_{raw,src}.csv
# Usage: tools/perf/ncu_seq_eval.sh [kernel-regex-name]
k=${1:-k_seq_eval}
ncu --set full --import-source on --clock-control none -k regex:$k -s 20 -c 1 -f -o /tmp/$k \
  python bench.py --config cfg4 --no-sub --no-e2e --no-cpu --steps 1 --warmup 3 --iters 10 > gpurun_out/${k}_ncu.log 2>&1
ncu -i /tmp/$k.ncu-rep --page raw --csv > gpurun_out/${k}_raw.csv
ncu -i /tmp/$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${k}_src.csv
tail -2 gpurun_out/${k}_ncu.log
