timeout 1200 python -m pytest tests/test_gpu_zoom.py tests/test_gpu_guards.py -x -q 2>&1 | tail -3
timeout 2400 python tools/sweep.py --out gpurun_out/r2_cfg5_sweep_v9.json > gpurun_out/r2_sweep_v9.log 2>&1
tail -2 gpurun_out/r2_sweep_v9.log | cut -c1-200
python bench.py > gpurun_out/r2_bench_late.json 2> gpurun_out/r2_bench_late.err; tail -c 600 gpurun_out/r2_bench_late.err
