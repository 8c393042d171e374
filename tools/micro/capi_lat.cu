// Single-call latency floor on this box: an empty launch + sync, a small H2D + sync, and the C ABI's
// single-trace calls (sk_fft_spectrum, sk_czt_spectrum, sk_zoom_spectrum) from C++ (no Python in the
// loop). build: see tools/gpu_lat.sh
#include <chrono>
#include <cmath>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "spectralkit.h"

__global__ void k_empty() {}

template <typename F> double time_us(F&& f, int reps = 2000) {
    for (int i = 0; i < 50; ++i) f();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

int main() {
    cudaFree(nullptr);
    void* d = nullptr;
    void* h = nullptr;
    cudaMalloc(&d, 1 << 20);
    cudaHostAlloc(&h, 1 << 20, cudaHostAllocDefault);
    printf("empty launch + sync: %.1f us\n", time_us([] { k_empty<<<1, 32>>>(); cudaDeviceSynchronize(); }));
    printf("H2D 8 KB + sync: %.1f us\n", time_us([&] {
               cudaMemcpyAsync(d, h, 8192, cudaMemcpyHostToDevice, cudaStreamPerThread);
               cudaStreamSynchronize(cudaStreamPerThread);
           }));
    printf("H2D 8 KB + launch + D2H 64 KB + sync: %.1f us\n", time_us([&] {
               cudaMemcpyAsync(d, h, 8192, cudaMemcpyHostToDevice, cudaStreamPerThread);
               k_empty<<<1, 32, 0, cudaStreamPerThread>>>();
               cudaMemcpyAsync(h, d, 65536, cudaMemcpyDeviceToHost, cudaStreamPerThread);
               cudaStreamSynchronize(cudaStreamPerThread);
           }));
    const double fs = 20e12;
    for (int n : {500, 1024, 4096}) {
        std::vector<double> x(n);
        for (int i = 0; i < n; ++i) x[i] = std::sin(0.01 * i) * std::exp(-1e-3 * i);
        sk_trace* t = nullptr;
        sk_trace_create(x.data(), (size_t)n, fs, 0.0, &t);
        const size_t len = n == 500 ? 4096 : 4 * (size_t)n;
        printf("n=%d sk_fft_spectrum(len %zu): %.1f us\n", n, len, time_us([&] {
                   sk_spectrum* s = nullptr;
                   sk_fft_spectrum(t, len, &s);
                   sk_spectrum_free(s);
               }));
        printf("n=%d sk_czt_spectrum(0.1-3 THz, 2048): %.1f us\n", n, time_us([&] {
                   sk_spectrum* s = nullptr;
                   sk_czt_spectrum(t, 0.1e12, 3e12, 2048, &s);
                   sk_spectrum_free(s);
               }));
        sk_zoom_options o;
        sk_zoom_options_defaults(&o);
        o.decimation = 8;
        o.num_taps = 65;
        sk_zoom_plan* zp = nullptr;
        if (sk_zoom_plan_create((size_t)n, 0.4e12, 1.2e12, fs, &o, &zp) == SK_OK) {
            printf("n=%d sk_zoom_spectrum(D 8): %.1f us\n", n, time_us([&] {
                       sk_spectrum* s = nullptr;
                       sk_zoom_spectrum(zp, t, &s);
                       sk_spectrum_free(s);
                   }));
            sk_zoom_plan_free(zp);
        } else {
            printf("zoom plan: %s\n", sk_last_error());
        }
        sk_trace_free(t);
    }
    return 0;
}
