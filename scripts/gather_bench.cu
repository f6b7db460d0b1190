// Microbenchmark: cp.async row-gather pipeline throughput on sm_100a (no MMA, no epilogue).
// 148 CTAs; NW producer warps gather 128 random rows x RB bytes per stage into an S-stage
// ring; one consumer thread waits "full" and releases "empty".  Variants:
//   mode 0: cp.async + cp.async.mbarrier.arrive.noinc
//   mode 1: ld.global.v4 into registers + st.shared + mbarrier.arrive (sync copies)
//   mode 2: like 0 but rows contiguous (no gather)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/gather_bench.cu -o scripts/gather_bench.bin
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool tw(uint32_t b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                 : "=r"(ok)
                 : "r"(b), "r"(ph)
                 : "memory");
    return ok;
}

template <int RB, int NW, int MODE>
__global__ void __launch_bounds__(NW * 32 + 32, 1) k(const char *__restrict__ F, const int *__restrict__ idx, int n_rows,
                                                    int steps, long long *out_cycles) {
    constexpr int S = 8;
    extern __shared__ __align__(1024) char ring_raw[];
    auto ring = reinterpret_cast<char (*)[128 * RB]>(ring_raw);
    __shared__ __align__(8) uint64_t full[S], empty[S];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[s])), "r"(NW * 32));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[s])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    long long t0 = clock64();
    constexpr int NQ = RB / 16;
    constexpr int Q = NQ < 4 ? NQ : 4;
    constexpr int RPI = 32 / Q;
    constexpr int ROWS_W = 128 / NW;
    constexpr int NB = ROWS_W / RPI > 0 ? ROWS_W / RPI : 1;
    constexpr int NT = NQ / Q;
    if (warp < NW) {
        const int r_in = lane % RPI, q_lane = lane / RPI;
        int s = 0;
        uint32_t ph = 0;
        for (int it = 0; it < steps; ++it) {
            while (!tw(su(&empty[s]), ph ^ 1)) {
            }
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const int r = warp * ROWS_W + b * RPI + r_in;
                const int g = MODE == 2 ? ((blockIdx.x * 977 + it * 128 + r) % n_rows)
                                        : idx[((size_t)blockIdx.x * steps + it) % 65536 * 128 + r];
                const char *src = F + (size_t)g * RB + q_lane * 16;
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    const uint32_t dst = su(&ring[s][r * RB + (q_lane + t * Q) * 16]);
                    if (MODE == 1) {
                        int4 v = *reinterpret_cast<const int4 *>(src + t * Q * 16);
                        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(v.x), "r"(v.y), "r"(v.z),
                                     "r"(v.w));
                    } else {
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + t * Q * 16));
                    }
                }
            }
            if (MODE == 1)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&full[s])) : "memory");
            else
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su(&full[s])) : "memory");
            if (++s == S) { s = 0; ph ^= 1; }
        }
        asm volatile("cp.async.wait_all;");
    } else if (lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int it = 0; it < steps; ++it) {
            while (!tw(su(&full[s]), ph)) {
            }
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
            if (++s == S) { s = 0; ph ^= 1; }
        }
        out_cycles[blockIdx.x] = clock64() - t0;
    }
}

template <int RB, int NW, int MODE>
void run(const char *F, const int *idx, int n_rows, long long *d_cyc, const char *name) {
    const int steps = 2000;
    const int smem = 8 * 128 * RB;
    cudaFuncSetAttribute(k<RB, NW, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<RB, NW, MODE><<<148, NW * 32 + 32, smem>>>(F, idx, n_rows, steps, d_cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<RB, NW, MODE><<<148, NW * 32 + 32, smem>>>(F, idx, n_rows, steps, d_cyc);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> cyc(148);
    cudaMemcpy(cyc.data(), d_cyc, 148 * 8, cudaMemcpyDeviceToHost);
    double bytes = 148.0 * steps * 128 * RB;
    printf("%-28s RB=%3d NW=%d: %7.1f us  %6.0f cycles/step  %7.1f GB/s  %s\n", name, RB, NW, ms * 1e3,
           (double)cyc[0] / steps, bytes / (ms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    const int n_rows = 100000;
    char *F;
    int *idx;
    long long *d_cyc;
    cudaMalloc(&F, (size_t)n_rows * 256);
    cudaMalloc(&idx, 65536 * 128 * 4);
    cudaMalloc(&d_cyc, 148 * 8);
    std::vector<int> h(65536 * 128);
    srand(1);
    for (auto &v : h) v = rand() % n_rows;
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(F, 1, (size_t)n_rows * 256);
    run<64, 8, 0>(F, idx, n_rows, d_cyc, "cp.async gather noinc");
    run<64, 4, 0>(F, idx, n_rows, d_cyc, "cp.async gather noinc");
    run<64, 8, 1>(F, idx, n_rows, d_cyc, "ld+st gather");
    run<64, 8, 2>(F, idx, n_rows, d_cyc, "cp.async contiguous");
    run<128, 8, 0>(F, idx, n_rows, d_cyc, "cp.async gather noinc");
    run<128, 8, 1>(F, idx, n_rows, d_cyc, "ld+st gather");
    run<32, 8, 0>(F, idx, n_rows, d_cyc, "cp.async gather noinc");
    return 0;
}
