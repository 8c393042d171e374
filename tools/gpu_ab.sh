# A/B timing of library builds (default + paper_2108_03948_b200/lib_alt/*), then the band GPU tests
set -x
for lib in default paper_2108_03948_b200/lib_alt/*/libspectralkit_b200.so; do
  if [ "$lib" = default ]; then timeout 300 python tools/cube_time.py 20; else SKG_LIB_PATH=$lib timeout 300 python tools/cube_time.py 20; fi
done
timeout 600 python -m pytest tests/test_gpu_band.py tests/test_gpu_transfer.py tests/test_gpu_fft.py -x -q 2>&1 | tail -15
