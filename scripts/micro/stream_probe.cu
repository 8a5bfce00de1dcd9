// Micro-probe (not product code): how fast can a 3.456M-element fp64
// gather-free stream y[j] = f(x[j]) run on this B200 at the size of the
// Goofspiel-5 deepest level, by launch shape and loads-in-flight per thread?
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a stream_probe.cu -o stream_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int IT>
__global__ void k_stride(const double* __restrict__ x, double* __restrict__ y, int n) {
    const int stride = gridDim.x * blockDim.x;
    for (int base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * IT) {
        double v[IT];
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const int k = base + i * stride;
            if (k < n) v[i] = x[k];
        }
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const int k = base + i * stride;
            if (k < n) y[k] = v[i] * 1.0 + 0.0;
        }
    }
}

__global__ void k_flat(const double* __restrict__ x, double* __restrict__ y, int n) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) y[k] = x[k] * 1.0 + 0.0;
}

__global__ void k_flush(double* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] += 1.0;
}

int main() {
    const int n = 3456000;
    double *x, *y, *junk;
    const size_t J = 64ull << 20;  // 512 MB: evicts L2
    cudaMalloc(&x, n * 8);
    cudaMalloc(&y, n * 8);
    cudaMalloc(&junk, J * 8);
    cudaMemset(x, 0, n * 8);
    cudaMemset(junk, 0, J * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time = [&](const char* name, auto launch, bool flush) {
        float best = 1e9, sum = 0;
        for (int r = 0; r < 20; ++r) {
            if (flush) k_flush<<<1184, 256>>>(junk, J);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 2) { best = ms < best ? ms : best; sum += ms; }
        }
        printf("%-34s %s best %7.2f us  mean %7.2f us  -> %6.0f GB/s (16 B/elem)\n", name, flush ? "cold" : "warm",
               best * 1e3, sum / 18 * 1e3, 16.0 * n / (best * 1e-3) / 1e9);
    };
    for (int flush = 1; flush >= 0; --flush) {
        time("flat 1 elem/thread (27k CTAs x128)", [&] { k_flat<<<(n + 127) / 128, 128>>>(x, y, n); }, flush);
        time("stride IT1 1776x128", [&] { k_stride<1><<<1776, 128>>>(x, y, n); }, flush);
        time("stride IT4 1776x128", [&] { k_stride<4><<<1776, 128>>>(x, y, n); }, flush);
        time("stride IT4 888x128", [&] { k_stride<4><<<888, 128>>>(x, y, n); }, flush);
        time("stride IT8 1184x256", [&] { k_stride<8><<<1184, 256>>>(x, y, n); }, flush);
        time("stride IT2 2368x256", [&] { k_stride<2><<<2368, 256>>>(x, y, n); }, flush);
    }
    return 0;
}
