# round 2: full-batch parity + the whole GPU suite + a bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_fullbatch.py -q -x --durations=15 > gpurun_out/pytest_full.log 2>&1; echo full_rc=$?
tail -30 gpurun_out/pytest_full.log
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo gpu_rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench.log
