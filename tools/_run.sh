timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
python bench.py > gpurun_out/r2_bench_late2.json 2> gpurun_out/r2_bench_late2.err; tail -c 300 gpurun_out/r2_bench_late2.err
