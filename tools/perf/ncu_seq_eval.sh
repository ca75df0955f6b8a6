#!/bin/bash
# ncu --set full of one warm k_seq_eval launch of the cfg4 fit (bench.py --config cfg4), exported
# as raw + SASS-source CSVs into gpurun_out/seqeval_{raw,src}.csv
ncu --set full --import-source on --clock-control none -k regex:k_seq_eval -s 20 -c 1 -f -o /tmp/seqeval \
  python bench.py --config cfg4 --no-sub --no-e2e --no-cpu --steps 1 --warmup 3 --iters 10 > gpurun_out/seqeval_ncu.log 2>&1
ncu -i /tmp/seqeval.ncu-rep --page raw --csv > gpurun_out/seqeval_raw.csv
ncu -i /tmp/seqeval.ncu-rep --page source --csv --print-source sass > gpurun_out/seqeval_src.csv
tail -2 gpurun_out/seqeval_ncu.log
