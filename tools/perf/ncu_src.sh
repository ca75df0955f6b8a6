#!/bin/bash
# ncu --set full of the timed k_fit launch of `bench.py --config $1 [extra flags]`, exported as
# raw + SASS-source CSVs into gpurun_out/<name>_{raw,src}.csv (the .ncu-rep stays in /tmp: too
# large for gpurun_out).  Usage: tools/perf/ncu_src.sh name config [bench flags...]
name=$1; cfg=$2; shift 2
ncu --set full --import-source on --clock-control none -k regex:k_fit -s 1 -c 1 -f -o /tmp/$name \
  python bench.py --config $cfg --no-sub --no-e2e --no-cpu --steps 1 --warmup 1 "$@" > gpurun_out/${name}_ncu.log 2>&1
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_src.csv
tail -2 gpurun_out/${name}_ncu.log
