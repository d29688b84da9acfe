// hop_bench.cu — one-hop latency of the LL neighbour exchange for store/load flavours.
// 148 CTAs on a ring, 256 threads; round r: poll both neighbours' cells of round r-1, then store own cells.
// Strict chain (D = 1): ns per round = one exchange hop.  SV = store flavour, LV = load flavour.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

template <int SV>
__device__ __forceinline__ void put(unsigned long long* p, unsigned long long w0, unsigned long long w1) {
    if (SV == 0) asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
    if (SV == 1) asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
    if (SV == 2) asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
    if (SV == 3) asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
    if (SV == 4) { asm volatile("atom.global.exch.b64 %0, [%1], %0;" : "+l"(w0) : "l"(p) : "memory");
                   asm volatile("atom.global.exch.b64 %0, [%1], %0;" : "+l"(w1) : "l"(p + 1) : "memory"); }
    if (SV == 5) asm volatile("st.global.cs.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
template <int LV>
__device__ __forceinline__ void get(const unsigned long long* p, unsigned long long& w0, unsigned long long& w1) {
    if (LV == 0) asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    if (LV == 1) asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    if (LV == 2) asm volatile("ld.global.cv.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    if (LV == 3) asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}

constexpr int R = 8, T = 256;
template <int SV, int LV>
__global__ void __launch_bounds__(T, 1) hop(unsigned long long* cells, int rounds, int nthr, double* out) {
    const int G = gridDim.x, c = blockIdx.x, t = threadIdx.x;
    const int cn = c + 1 == G ? 0 : c + 1, cs = c == 0 ? G - 1 : c - 1;
    double acc = 0;
    for (int r = 0; r < rounds; ++r) {
        if (r > 0 && t < nthr) {
            const unsigned f = r;   // neighbours' round r-1 has flag r
            for (int side = 0; side < 2; ++side) {
                const int nb = side ? cn : cs;
                const unsigned long long* p = cells + ((((size_t)nb * R + (r - 1) % R) * 2 + (1 - side)) * T + t) * 2;
                unsigned long long w0, w1;
                do { get<LV>(p, w0, w1); } while ((unsigned)(w0 >> 32) != f || (unsigned)(w1 >> 32) != f);
                acc += (double)(unsigned)w0;
            }
        }
        __syncwarp();
        if (t < nthr) {
            const unsigned long long w = ((unsigned long long)(r + 1) << 32) | (unsigned)r;
            for (int side = 0; side < 2; ++side)
                put<SV>(cells + ((((size_t)c * R + r % R) * 2 + side) * T + t) * 2, w, w);
        }
    }
    if (acc == 1.5) out[0] = acc;
}

template <int SV, int LV>
float run(int G, int rounds, int nthr, unsigned long long* cells, double* out) {
    cudaMemset(cells, 0, (size_t)G * R * 2 * T * 16);
    void* args[] = {&cells, &rounds, &nthr, &out};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)hop<SV, LV>, G, T, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (cudaGetLastError() != cudaSuccess) { printf("err\n"); exit(1); }
    return ms * 1e6f / rounds;
}

int main() {
    int G = 0;
    cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* cells; double* out;
    cudaMalloc(&cells, (size_t)G * R * 2 * T * 16);
    cudaMalloc(&out, 8);
    const int rounds = 20000;
    const char* sn[] = {"st.wb", "st.cg", "st.relaxed.gpu", "st.volatile", "atom.exch", "st.cs"};
    const char* ln[] = {"ld.relaxed.gpu", "ld.volatile", "ld.cv", "ld.cg"};
    for (int nthr : {256, 32}) {
        printf("threads exchanging per CTA: %d  (ns per hop)\n", nthr);
        float v[6][4];
        v[0][0] = run<0, 0>(G, rounds, nthr, cells, out); v[0][1] = run<0, 1>(G, rounds, nthr, cells, out);
        v[0][2] = run<0, 2>(G, rounds, nthr, cells, out); v[0][3] = run<0, 3>(G, rounds, nthr, cells, out);
        v[1][0] = run<1, 0>(G, rounds, nthr, cells, out); v[1][1] = run<1, 1>(G, rounds, nthr, cells, out);
        v[2][0] = run<2, 0>(G, rounds, nthr, cells, out); v[2][1] = run<2, 1>(G, rounds, nthr, cells, out);
        v[3][0] = run<3, 0>(G, rounds, nthr, cells, out); v[3][1] = run<3, 1>(G, rounds, nthr, cells, out);
        v[4][0] = run<4, 0>(G, rounds, nthr, cells, out); v[4][1] = run<4, 1>(G, rounds, nthr, cells, out);
        v[5][0] = run<5, 0>(G, rounds, nthr, cells, out); v[5][1] = run<5, 1>(G, rounds, nthr, cells, out);
        for (int s = 0; s < 6; ++s)
            printf("  %-16s %s %7.0f   %s %7.0f%s\n", sn[s], ln[0], v[s][0], ln[1], v[s][1],
                   s == 0 ? "" : "");
        printf("  st.wb + ld.cv %7.0f   st.wb + ld.cg %7.0f\n", v[0][2], v[0][3]);
    }
    return 0;
}
