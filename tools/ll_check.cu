// ll_check.cu — correctness of the LL poll for load flavours: every consumed value must equal what the producer
// wrote under the matching flag (counts mismatches).  Same ring as hop_bench.cu.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
constexpr int R = 8, T = 256;
template <int LV>
__device__ __forceinline__ void get(const unsigned long long* p, unsigned long long& w0, unsigned long long& w1) {
    if (LV == 0) asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    if (LV == 1) asm volatile("ld.global.cv.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    if (LV == 2) asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    if (LV == 3) { asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(w0) : "l"(p) : "memory");
                   asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(w1) : "l"(p + 1) : "memory"); }
    if (LV == 4) { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w0) : "l"(p) : "memory");
                   asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w1) : "l"(p + 1) : "memory"); }
}
template <int LV>
__global__ void __launch_bounds__(T, 1) chk(unsigned long long* cells, int rounds, unsigned* bad) {
    const int G = gridDim.x, c = blockIdx.x, t = threadIdx.x;
    const int cn = c + 1 == G ? 0 : c + 1, cs = c == 0 ? G - 1 : c - 1;
    unsigned nbad = 0;
    for (int r = 0; r < rounds; ++r) {
        if (r > 0) {
            const unsigned f = r;
            for (int side = 0; side < 2; ++side) {
                const int nb = side ? cn : cs;
                const unsigned long long* p = cells + ((((size_t)nb * R + (r - 1) % R) * 2 + (1 - side)) * T + t) * 2;
                unsigned long long w0, w1;
                do { get<LV>(p, w0, w1); } while ((unsigned)(w0 >> 32) != f || (unsigned)(w1 >> 32) != f);
                const unsigned want0 = (unsigned)(nb * 1000003u + t * 7919u + (r - 1) * 31u + (1 - side));
                if ((unsigned)w0 != want0 || (unsigned)w1 != ~want0) ++nbad;
            }
        }
        for (int side = 0; side < 2; ++side) {
            const unsigned v = (unsigned)(c * 1000003u + t * 7919u + r * 31u + side);
            const unsigned long long w0 = ((unsigned long long)(r + 1) << 32) | v, w1 = ((unsigned long long)(r + 1) << 32) | ~v;
            asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(cells + ((((size_t)c * R + r % R) * 2 + side) * T + t) * 2), "l"(w0), "l"(w1) : "memory");
        }
    }
    atomicAdd(bad, nbad);
}
template <int LV>
unsigned run(int G, unsigned long long* cells, unsigned* bad, float* ns) {
    const int rounds = 20000;
    cudaMemset(cells, 0, (size_t)G * R * 2 * T * 16);
    cudaMemset(bad, 0, 4);
    void* args[] = {&cells, (void*)&rounds, &bad};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)chk<LV>, G, T, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); *ns = ms * 1e6f / rounds;
    unsigned h; cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
    return h;
}
int main() {
    int G; cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* cells; unsigned* bad;
    cudaMalloc(&cells, (size_t)G * R * 2 * T * 16); cudaMalloc(&bad, 4);
    const char* n[] = {"ld.relaxed.gpu.v2", "ld.cv.v2", "ld.cg.v2", "ld.cv x2 (u64)", "ld.relaxed.gpu x2 (u64)"};
    float ns; unsigned b;
    b = run<0>(G, cells, bad, &ns); printf("%-26s mismatches %u  %.0f ns/hop\n", n[0], b, ns);
    b = run<1>(G, cells, bad, &ns); printf("%-26s mismatches %u  %.0f ns/hop\n", n[1], b, ns);
    b = run<2>(G, cells, bad, &ns); printf("%-26s mismatches %u  %.0f ns/hop\n", n[2], b, ns);
    b = run<3>(G, cells, bad, &ns); printf("%-26s mismatches %u  %.0f ns/hop\n", n[3], b, ns);
    b = run<4>(G, cells, bad, &ns); printf("%-26s mismatches %u  %.0f ns/hop\n", n[4], b, ns);
    return 0;
}
