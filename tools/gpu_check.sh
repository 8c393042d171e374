timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_io.py tests/test_gpu_band.py -q > gpurun_out/pytest_gpu3.log 2>&1; tail -30 gpurun_out/pytest_gpu3.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench3.log 2> gpurun_out/bench3.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench3.log').read().strip().splitlines()[-1])
print(json.dumps({k: d['extra'][k] for k in ('csv_pipeline_f64','resolvability_scan_thz','cfg4_cube_H_f32')}, indent=1))"
tail -5 gpurun_out/bench3.err
