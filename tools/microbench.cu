// microbench.cu — box constants that decide the solver design:
//   1. grid-barrier latency (cooperative, G = SMs x occ) for two barrier implementations
//   2. fp64 FMA peak (the "alu" roofline denominator of the level solves)
//   3. L2-resident read bandwidth (working set 32 MB) and HBM copy bandwidth (2 GB)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}

// A: counter + generation (reset by the last arriver)
__global__ void bar_gen(unsigned* w, int iters) {
    unsigned gen = 0;
    if (threadIdx.x == 0) gen = ld_acq(&w[1]);
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            unsigned a = atomicAdd(&w[0], 1u);
            if (a == gridDim.x - 1) { atomicExch(&w[0], 0u); __threadfence(); atomicExch(&w[1], gen + 1); }
            else while (ld_acq(&w[1]) == gen) {}
            __threadfence();
            gen++;
        }
        __syncthreads();
    }
}

// B: monotonic counter, red.release + ld.acquire spin (no reset, one atomic per CTA)
__global__ void bar_mono(unsigned* w, int iters) {
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned target = (unsigned)(i + 1) * gridDim.x;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(w) : "memory");
            while (ld_acq(w) < target) {}
        }
        __syncthreads();
    }
}

__global__ void fma_peak(double* out, int iters) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
        #pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 12345.0) out[0] = 1;
}

__global__ void read_sum(const double2* __restrict__ x, size_t n, int reps, double* out) {
    double s = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            double2 v = x[i]; s += v.x + v.y;
        }
    if (s == 1234.5) out[0] = s;
}

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
    cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
    const int sms = pr.multiProcessorCount;
    printf("device %s, %d SMs, clock %d kHz\n", pr.name, sms, pr.clockRate);
    unsigned* w; CK(cudaMalloc(&w, 64));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int occ = 1; occ <= 2; ++occ) {
        for (int kind = 0; kind < 2; ++kind) {
            int iters = 20000;
            int G = sms * occ;
            void* args[] = {&w, &iters};
            CK(cudaMemset(w, 0, 64));
            CK(cudaLaunchCooperativeKernel(kind ? (void*)bar_mono : (void*)bar_gen, G, 256, args, 0, 0));
            CK(cudaDeviceSynchronize());
            CK(cudaMemset(w, 0, 64));
            cudaEventRecord(e0);
            CK(cudaLaunchCooperativeKernel(kind ? (void*)bar_mono : (void*)bar_gen, G, 256, args, 0, 0));
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("grid barrier %-4s G=%d: %.3f us per barrier\n", kind ? "mono" : "gen", G, ms * 1e3 / iters);
        }
    }
    double* out; CK(cudaMalloc(&out, 8));
    {
        int iters = 20000; int G = sms * 8;
        fma_peak<<<G, 256>>>(out, 10); CK(cudaDeviceSynchronize());
        cudaEventRecord(e0); fma_peak<<<G, 256>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 16 * (double)iters * G * 256;
        printf("fp64 FMA: %.2f TFLOP/s\n", flops / (ms * 1e-3) / 1e12);
    }
    {
        size_t bytes = 32ull << 20; size_t n = bytes / 16; double2* x; CK(cudaMalloc(&x, bytes)); CK(cudaMemset(x, 0, bytes));
        int reps = 50;
        read_sum<<<sms * 8, 256>>>(x, n, 2, out); CK(cudaDeviceSynchronize());
        cudaEventRecord(e0); read_sum<<<sms * 8, 256>>>(x, n, reps, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("L2-resident read (32 MB x %d): %.0f GB/s\n", reps, (double)bytes * reps / (ms * 1e-3) / 1e9);
        cudaFree(x);
    }
    {
        size_t bytes = 2ull << 30; size_t n = bytes / 16; double2 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
        CK(cudaMemset(a, 0, bytes));
        copy_k<<<sms * 8, 256>>>(a, b, n); CK(cudaDeviceSynchronize());
        cudaEventRecord(e0); for (int r = 0; r < 5; ++r) copy_k<<<sms * 8, 256>>>(a, b, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("HBM copy 2 GB (read+write): %.0f GB/s\n", 2.0 * bytes * 5 / (ms * 1e-3) / 1e9);
    }
    return 0;
}
