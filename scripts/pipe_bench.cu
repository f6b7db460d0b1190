// Microbenchmark: cp.async row gather -> tcgen05.mma pipeline (no scheduler, no epilogue).
// 148 CTAs x (8 gather warps + 1 MMA warp).  Stage = ROWS x 32 bf16 (64-B rows, SWIZZLE_64B),
// weight tile N x 32 static in smem.  Variants of the consumer:
//   C=0: wait full, arrive empty (no MMA)            C=1: + fence.proxy.async
//   C=2: + tcgen05.mma x (ROWS/128)*2, commit->empty  C=3: MMA without the proxy fence
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/pipe_bench.cu -o scripts/pipe_bench.bin
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
__device__ __forceinline__ uint64_t desc64(uint32_t addr) {   // K-major SWIZZLE_64B, rb = 64
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((512 >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}

template <int ROWS, int C, int REAL_PCT>
__global__ void __launch_bounds__(288, 1) k(const char *__restrict__ F, const int *__restrict__ idx, int n_rows,
                                            int steps, long long *out_cycles) {
    constexpr int S = 8, RB = 64, N = 96;
    extern __shared__ __align__(1024) char smem_raw[];
    char *ring = smem_raw;                               // S x ROWS x 64
    char *wtile = smem_raw + S * ROWS * RB;              // N x 64
    __shared__ __align__(8) uint64_t full[S], empty[S];
    __shared__ uint32_t tmem_hold;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[s])), "r"(256));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[s])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int i = threadIdx.x; i < N * RB / 4; i += blockDim.x) reinterpret_cast<int *>(wtile)[i] = 0;
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&tmem_hold)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_hold;
    long long t0 = clock64();
    if (warp < 8) {
        constexpr int Q = 4, RPI = 8, ROWS_W = ROWS / 8, NB = ROWS_W / RPI;
        const int r_in = lane % RPI, q_lane = lane / RPI;
        int s = 0;
        uint32_t ph = 0;
        for (int it = 0; it < steps; ++it) {
            while (!tw(su(&empty[s]), ph ^ 1)) {
            }
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const int r = warp * ROWS_W + b * RPI + r_in;
                const int g = idx[((size_t)blockIdx.x * steps + it) % 65536 * 128 + (r & 127)];
                const uint32_t f = (r >> 1) & 3;
                const uint32_t dst = su(ring + s * ROWS * RB + r * RB + ((q_lane ^ f) * 16));
                if ((g % 100) < REAL_PCT)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                                 "l"(F + (size_t)g * RB + q_lane * 16));
                else
                    asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(dst), "r"(0) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su(&full[s])) : "memory");
            if (++s == S) { s = 0; ph ^= 1; }
        }
        asm volatile("cp.async.wait_all;");
    } else if (lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        for (int it = 0; it < steps; ++it) {
            while (!tw(su(&full[s]), ph)) {
            }
            if (C == 1 || C == 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (C >= 2) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t a0 = su(ring + s * ROWS * RB), b0 = su(wtile);
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                    for (int h = 0; h < ROWS / 128; ++h) {
                        const uint64_t ad = desc64(a0 + h * 128 * RB + kk * 32), bd = desc64(b0 + kk * 32);
                        const uint32_t acc = (it | kk) ? 1u : 0u;
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, "
                            "%3, p;\n}" ::"r"(tmem + h * 128),
                            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                    }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 su(&empty[s]))
                             : "memory");
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
            }
            if (++s == S) { s = 0; ph ^= 1; }
        }
        out_cycles[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 8) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    }
}

template <int ROWS, int C, int REAL>
void run(const char *F, const int *idx, int n_rows, long long *d_cyc) {
    const int steps = 2000;
    const int smem = 8 * ROWS * 64 + 96 * 64 + 1024;
    cudaFuncSetAttribute(k<ROWS, C, REAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<ROWS, C, REAL><<<148, 288, smem>>>(F, idx, n_rows, steps, d_cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<ROWS, C, REAL><<<148, 288, smem>>>(F, idx, n_rows, steps, d_cyc);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> cyc(148);
    cudaMemcpy(cyc.data(), d_cyc, 148 * 8, cudaMemcpyDeviceToHost);
    printf("rows=%d consumer=%d real=%3d%%: %7.1f us  %6.0f cycles/step %s\n", ROWS, C, REAL, ms * 1e3,
           (double)cyc[0] / steps, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    const int n_rows = 100000;
    char *F;
    int *idx;
    long long *d_cyc;
    cudaMalloc(&F, (size_t)n_rows * 64);
    cudaMalloc(&idx, 65536 * 128 * 4);
    cudaMalloc(&d_cyc, 148 * 8);
    std::vector<int> h(65536 * 128);
    srand(1);
    for (auto &v : h) v = rand() % n_rows;
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(F, 1, (size_t)n_rows * 64);
    run<128, 0, 100>(F, idx, n_rows, d_cyc);
    run<128, 1, 100>(F, idx, n_rows, d_cyc);
    run<128, 2, 100>(F, idx, n_rows, d_cyc);
    run<128, 3, 100>(F, idx, n_rows, d_cyc);
    run<128, 2, 22>(F, idx, n_rows, d_cyc);
    run<256, 0, 22>(F, idx, n_rows, d_cyc);
    run<256, 2, 22>(F, idx, n_rows, d_cyc);
    run<256, 2, 100>(F, idx, n_rows, d_cyc);
    return 0;
}
