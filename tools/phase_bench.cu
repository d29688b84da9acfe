// phase_bench.cu — cost model of one BiCGSTAB phase of the column-blocked engine, in isolation.
// 148 CTAs x 512 threads, each thread a column of H rows (c5 at D = 2: H = 7), u / operand / v / t in shared
// memory, sr / pp in registers.  Variants (argv[1]):
//   0: full phase = halo L2 loads + s update + sync + matvec + 5 dots + block reduce + partial store +
//      grid barrier + pair reduce (L2 round trip)
//   1: no grid barrier / pair reduce (CTA-local phase work only)
//   2: variant 1 without the halo loads
//   3: variant 2 without the block reduce
//   4: barrier + pair reduce only (no work)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o phase_bench phase_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

constexpr int NT = 512, H = 7, NX = 512, W = NX + 2;

__device__ __forceinline__ unsigned ld_acq(const unsigned long long* p, unsigned long long& v) {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return 0;
}

template <int VAR>
__global__ void __launch_bounds__(NT, 1) phase(double* gpub, double* part, unsigned long long* ctr, int iters, double* out) {
    extern __shared__ double sm[];
    double* u_s = sm;                  // (H+2) x W
    double* op_s = u_s + (H + 2) * W;  // (H+2) x W
    double* v_s = op_s + (H + 2) * W;  // H x NT
    double* t_s = v_s + H * NT;
    double* bt_s = t_s + H * NT;
    __shared__ double red[NT / 32 * 5];
    __shared__ double pr[8];
    const int tid = threadIdx.x, col = tid;
    for (int i = tid; i < (H + 2) * W; i += NT) { u_s[i] = 0.1 * (i % 7); op_s[i] = 0.0; }
    for (int i = tid; i < H * NT; i += NT) { v_s[i] = 1e-3 * (i % 5); bt_s[i] = 1.0; t_s[i] = 0.0; }
    double sr[H];
    #pragma unroll
    for (int r = 0; r < H; ++r) sr[r] = 0.01 * (r + 1);
    __syncthreads();
    const double alpha = 0.5, cx = 0.0256, dx = 0.131, ci = 0.656;
    double acc = 0.0;
    unsigned long long target = 0;
    for (int itn = 0; itn < iters; ++itn) {
        double a[5] = {0, 0, 0, 0, 0};
        double hS0 = 0, hS1 = 0, hN0 = 0, hN1 = 0;
        if (VAR <= 1 || VAR >= 5) {
            hS0 = __ldcg(gpub + ((blockIdx.x + 1) % gridDim.x) * NX + col);
            hS1 = __ldcg(gpub + ((blockIdx.x + 2) % gridDim.x) * NX + col);
            hN0 = __ldcg(gpub + ((blockIdx.x + 3) % gridDim.x) * NX + col);
            hN1 = __ldcg(gpub + ((blockIdx.x + 4) % gridDim.x) * NX + col);
        }
        if (VAR != 4 && VAR != 7) {
            #pragma unroll
            for (int r = 0; r < H; ++r) {
                const double s = sr[r] - alpha * v_s[r * NT + tid];
                sr[r] = s;
                op_s[(r + 1) * W + col + 1] = s;
                if (col == 0) op_s[(r + 1) * W + NX + 1] = s;
                if (col == NX - 1) op_s[(r + 1) * W] = s;
            }
            const double haloS = hS0 - alpha * hS1, haloN = hN0 - alpha * hN1;
            __syncthreads();
            #pragma unroll
            for (int r = 0; r < H; ++r) {
                const int si = (r + 1) * W + col + 1;
                const double e = cx * u_s[si + 1] - dx, w = -cx * u_s[si - 1] - dx;
                const double n = cx * u_s[si + W] - dx, s_ = -cx * u_s[si - W] - dx;
                const double on = r + 1 < H ? sr[r + 1] : haloN, os = r > 0 ? sr[r - 1] : haloS;
                const double sv = sr[r];
                const double t = sv + ci * (e * op_s[si + 1] + w * op_s[si - 1] + n * on + s_ * os);
                t_s[r * NT + tid] = t;
                const double b0 = bt_s[r * NT + tid];
                a[0] += t * sv; a[1] += t * t; a[2] += b0 * sv; a[3] += b0 * t; a[4] += sv * sv;
            }
            if (VAR == 5) {
                // streamlined: warp butterfly -> smem -> ONE __syncthreads -> warp 0 reduces, thread 0 publishes +
                // arrives + spins, warp 0 pair-reduces from L2, ONE __syncthreads broadcasts
                #pragma unroll
                for (int i = 0; i < 5; ++i)
                    #pragma unroll
                    for (int o = 16; o > 0; o >>= 1) a[i] += __shfl_xor_sync(0xffffffffu, a[i], o);
                if ((tid & 31) == 0) for (int i = 0; i < 5; ++i) red[(tid >> 5) * 5 + i] = a[i];
                __syncthreads();
                if (tid < 32) {
                    #pragma unroll
                    for (int i = 0; i < 5; ++i) {
                        double v = tid < NT / 32 ? red[tid * 5 + i] : 0.0;
                        #pragma unroll
                        for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                        a[i] = v;
                    }
                    if (tid == 0) {
                        for (int i = 0; i < 5; ++i) part[blockIdx.x * 8 + i] = a[i];
                        target += gridDim.x;
                        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
                        unsigned long long v;
                        do { ld_acq(ctr, v); } while (v < target);
                    }
                    __syncwarp();
                    const int g0 = blockIdx.x < 74 ? 0 : 74;
                    double y[5] = {0, 0, 0, 0, 0};
                    double ld[3][5];
                    #pragma unroll
                    for (int j = 0; j < 3; ++j)
                        #pragma unroll
                        for (int i = 0; i < 5; ++i) ld[j][i] = tid + 32 * j < 74 ? __ldcg(part + (g0 + tid + 32 * j) * 8 + i) : 0.0;
                    #pragma unroll
                    for (int j = 0; j < 3; ++j)
                        #pragma unroll
                        for (int i = 0; i < 5; ++i) y[i] += ld[j][i];
                    #pragma unroll
                    for (int i = 0; i < 5; ++i)
                        #pragma unroll
                        for (int o = 16; o > 0; o >>= 1) y[i] += __shfl_xor_sync(0xffffffffu, y[i], o);
                    if (tid < 5) pr[tid] = y[0] + y[1] + y[2] + y[3] + y[4];
                }
                __syncthreads();
                acc += pr[0] + pr[4];
            }
            if (VAR == 6) {
                // LL-flagged partials: no counter; readers poll the pair's slots (value halves + epoch flags in
                // 8-byte words), one L2 round trip after the last writer
                #pragma unroll
                for (int i = 0; i < 5; ++i)
                    #pragma unroll
                    for (int o = 16; o > 0; o >>= 1) a[i] += __shfl_xor_sync(0xffffffffu, a[i], o);
                if ((tid & 31) == 0) for (int i = 0; i < 5; ++i) red[(tid >> 5) * 5 + i] = a[i];
                __syncthreads();
                if (tid < 32) {
                    #pragma unroll
                    for (int i = 0; i < 5; ++i) {
                        double v = tid < NT / 32 ? red[tid * 5 + i] : 0.0;
                        #pragma unroll
                        for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                        a[i] = v;
                    }
                    const unsigned ep = (unsigned)itn + 1u;
                    uint4* slots = reinterpret_cast<uint4*>(part) + (size_t)(ep & 1u) * gridDim.x * 5;
                    if (tid == 0) {
                        asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        #pragma unroll
                        for (int i = 0; i < 5; ++i) {
                            const unsigned long long b = __double_as_longlong(a[i]);
                            asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(slots + blockIdx.x * 5 + i),
                                         "r"((unsigned)b), "r"(ep), "r"((unsigned)(b >> 32)), "r"(ep) : "memory");
                        }
                    }
                    const int g0 = blockIdx.x < 74 ? 0 : 74;
                    double y[5] = {0, 0, 0, 0, 0};
                    uint4 q[3][5];
                    for (;;) {
                        bool ok = true;
                        #pragma unroll
                        for (int j = 0; j < 3; ++j)
                            #pragma unroll
                            for (int i = 0; i < 5; ++i) {
                                if (tid + 32 * j < 74) {
                                    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                                                 : "=r"(q[j][i].x), "=r"(q[j][i].y), "=r"(q[j][i].z), "=r"(q[j][i].w)
                                                 : "l"(slots + (g0 + tid + 32 * j) * 5 + i) : "memory");
                                    ok = ok && q[j][i].y == ep && q[j][i].w == ep;
                                } else {
                                    q[j][i] = make_uint4(0, ep, 0, ep);
                                }
                            }
                        if (__all_sync(0xffffffffu, ok)) break;
                    }
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    #pragma unroll
                    for (int j = 0; j < 3; ++j)
                        #pragma unroll
                        for (int i = 0; i < 5; ++i)
                            y[i] += __longlong_as_double(((long long)q[j][i].z << 32) | q[j][i].x);
                    #pragma unroll
                    for (int i = 0; i < 5; ++i)
                        #pragma unroll
                        for (int o = 16; o > 0; o >>= 1) y[i] += __shfl_xor_sync(0xffffffffu, y[i], o);
                    if (tid < 5) pr[tid] = y[0] + y[1] + y[2] + y[3] + y[4];
                }
                __syncthreads();
                acc += pr[0] + pr[4];
            }
            if (VAR <= 2) {
                #pragma unroll
                for (int i = 0; i < 5; ++i)
                    #pragma unroll
                    for (int o = 16; o > 0; o >>= 1) a[i] += __shfl_xor_sync(0xffffffffu, a[i], o);
                if ((tid & 31) == 0) for (int i = 0; i < 5; ++i) red[(tid >> 5) * 5 + i] = a[i];
                __syncthreads();
                if (tid < 32) {
                    #pragma unroll
                    for (int i = 0; i < 5; ++i) {
                        double v = tid < NT / 32 ? red[tid * 5 + i] : 0.0;
                        #pragma unroll
                        for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                        a[i] = v;
                    }
                }
                __syncthreads();
                if (tid == 0) for (int i = 0; i < 5; ++i) part[blockIdx.x * 8 + i] = a[i];
            }
        }
        if (VAR == 0 || VAR == 4 || VAR == 7) {
            __syncthreads();
            if (tid == 0) {
                unsigned long long* c = VAR == 7 ? ctr + 16 * (blockIdx.x < 74 ? 0 : 1) : ctr;
                target += VAR == 7 ? 74 : gridDim.x;
                asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(c) : "memory");
                unsigned long long v;
                do { ld_acq(c, v); } while (v < target);
            }
            if (false) {
                unsigned long long v;
                do { ld_acq(ctr, v); } while (v < target);
            }
            __syncthreads();
            // pair reduce over 74 CTAs
            const int g0 = blockIdx.x < 74 ? 0 : 74;
            if (tid < 74) pr[0] = 0;  // placeholder staging
            double y = tid < 74 ? __ldcg(part + (g0 + tid) * 8) : 0.0;
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
            if ((tid & 31) == 0 && tid < 96) red[tid >> 5] = y;
            __syncthreads();
            acc += red[0] + red[1] + red[2];
            __syncthreads();
        }
        acc += sr[0];
    }
    if (acc == 1234.5) out[0] = acc;
}

int main(int argc, char** argv) {
    const int var = argc > 1 ? atoi(argv[1]) : 0;
    const int iters = 2000, G = 148;
    double *gpub, *part, *out;
    unsigned long long* ctr;
    cudaMalloc(&gpub, G * NX * 8); cudaMemset(gpub, 0, G * NX * 8);
    cudaMalloc(&part, G * 16 * 16); cudaMemset(part, 0, G * 256);
    cudaMalloc(&out, 8); cudaMalloc(&ctr, 256);
    const size_t smem = (size_t)(2 * (H + 2) * W + 3 * H * NT) * 8;
    void* fns[8] = {(void*)phase<0>, (void*)phase<1>, (void*)phase<2>, (void*)phase<3>, (void*)phase<4>, (void*)phase<5>, (void*)phase<6>, (void*)phase<7>};
    for (int v = 0; v < 8; ++v) cudaFuncSetAttribute(fns[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int v = (var >= 0 ? 0 : 0); v < 8; ++v) {
        int it = iters;
        void* args[] = {&gpub, &part, &ctr, &it, &out};
        cudaMemset(ctr, 0, 256); cudaMemset(part, 0, G * 256);
        cudaLaunchCooperativeKernel(fns[v], G, NT, args, smem, 0);
        cudaDeviceSynchronize();
        cudaMemset(ctr, 0, 256); cudaMemset(part, 0, G * 256);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel(fns[v], G, NT, args, smem, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("variant %d: %.3f us per phase (%s)\n", v, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
