# Round-end style validation on one B200: GPU tests, smoke, default bench, cfg4 bench, and the
# ncu launch list of the default bench command (gpu__time_duration per launch).
set -x
python -m pytest tests -m gpu -q > gpurun_out/fv_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fv_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fv_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fv_smoke.log
python bench.py > gpurun_out/fv_bench.log 2>&1; echo "rc=$?" >> gpurun_out/fv_bench.log
python bench.py --config cfg4 > gpurun_out/fv_bench_cfg4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fv_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --windows 131072 > gpurun_out/fv_ncu.log 2>&1
