# single-call latency floor + C ABI single-trace calls (C++ caller)
set -e
nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -Iinclude -o /tmp/capi_lat tools/micro/capi_lat.cu \
  -Lpaper_2108_03948_b200/lib -lspectralkit_b200 -Xlinker -rpath,$PWD/paper_2108_03948_b200/lib
/tmp/capi_lat
