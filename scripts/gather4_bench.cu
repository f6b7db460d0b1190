// Microbenchmark: row-gather throughput per SM on sm_100a, the A-operand feed of the OS
// feature kernel.  148 CTAs (one per SM), each gathering 128-row x 128-byte stages of
// random feature rows (bf16, 256 channels -> 512 B rows; one 64-channel chunk per row)
// into a ring of S stages, with a fraction of sentinel rows (-1):
//   mode 0: cp.async 16 B (LDGSTS) by 8 warps, sentinels zero-filled with st.shared
//   mode 1: TMA tile::gather4 (cp.async.bulk.tensor.2d ... gather4), 32 instructions per
//           stage issued by the 32 lanes of one warp; sentinels = out-of-range row -> zeros
// Reports bytes / cycle / SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// scripts/gather4_bench.cu -o gpurun_out/gather4_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int ROWS = 128, RB = 128, STAGE = ROWS * RB, S = 8;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                 : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
    return ok;
}

template <int MODE>
__global__ void __launch_bounds__(288, 1) k(const __grid_constant__ CUtensorMap tm, const char *F, int64_t ld,
                                            const int *idx, int n_idx, int iters, long long *cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + S * STAGE);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(MODE == 0 ? 256 : 1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const long long t0 = clock64();
    int base = (blockIdx.x * 7919) % n_idx;
    for (int it = 0; it < iters; ++it) {
        const int s = it % S;
        const uint32_t ph = (it / S) & 1;
        // the slot's previous fill must have landed (a consumer would release it here)
        if (it >= S) {
            if (MODE == 0 ? warp < 8 : warp == 8)
                while (!try_wait(smem_u32(&full[s]), ph ^ 1)) {}
        }
        const uint32_t dst = smem_u32(sm + s * STAGE);
        const int *ix = idx + (base + it * ROWS) % (n_idx - ROWS);
        if (MODE == 0) {
            if (warp < 8) {
                // 8 warps x 16 rows; lane -> (row within 4-row block, 16-byte chunk)
                const int r_in = lane >> 3, q = lane & 7;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int r = warp * 16 + b * 4 + r_in;
                    const int g = ix[r];
                    const uint32_t so = dst + r * RB + ((q ^ (r & 7)) * 16);
                    if (g >= 0)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(so), "l"(F + (int64_t)g * ld + q * 16)
                                     : "memory");
                    else
                        asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(so), "r"(0) : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
            }
        } else {
            if (warp == 8) {
                const uint32_t fb = smem_u32(&full[s]);
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(STAGE) : "memory");
                __syncwarp();
                const int r0 = lane * 4;
                int g[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) g[j] = ix[r0 + j];
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                    "%3, %4, %5, %6}], [%7];" ::"r"(dst + r0 * RB),
                    "l"(&tm), "r"(0), "r"(g[0]), "r"(g[1]), "r"(g[2]), "r"(g[3]), "r"(fb)
                    : "memory");
            }
        }
    }
    // drain
    for (int it = iters; it < iters + S; ++it) {
        const int s = it % S;
        if (it >= S && (MODE == 0 ? warp < 8 : warp == 8))
            while (!try_wait(smem_u32(&full[s]), ((it / S) & 1) ^ 1)) {}
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char **argv) {
    const double sent = argc > 1 ? atof(argv[1]) : 0.5;
    const int N = 100000, C = 256, iters = 2000;
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    char *F;
    cudaMalloc(&F, (size_t)N * C * 2);
    cudaMemset(F, 1, (size_t)N * C * 2);
    const int n_idx = 1 << 20;
    std::vector<int> h(n_idx);
    srand(1);
    for (auto &v : h) v = (rand() / (double)RAND_MAX) < sent ? -1 : rand() % N;
    int *idx;
    cudaMalloc(&idx, n_idx * 4);
    cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice);
    long long *cyc;
    cudaMalloc(&cyc, 148 * 8);
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)C, (cuuint64_t)N};
    cuuint64_t gstr[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, 1};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, F, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = S * STAGE + 1024;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 2; ++mode)
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148, 288, smem>>>(tm, F, C * 2, idx, n_idx, iters, cyc);
            else k<1><<<148, 288, smem>>>(tm, F, C * 2, idx, n_idx, iters, cyc);
            cudaEventRecord(b);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            std::vector<long long> c(148);
            cudaMemcpy(c.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (auto v : c) avg += v;
            avg /= 148;
            const double bytes = (double)iters * STAGE;   // per SM, sentinel rows included
            printf("mode %d (%s) sentinel %.2f: %.1f cycles/stage, %.1f B/clk/SM (all rows), %.1f B/clk/SM fetched; "
                   "%.3f ms, %.2f TB/s chip (all rows)\n",
                   mode, mode == 0 ? "cp.async" : "gather4", sent, avg / iters, bytes / avg, bytes * (1 - sent) / avg, ms,
                   bytes * 148 / (ms * 1e-3) / 1e12);
        }
    return 0;
}
