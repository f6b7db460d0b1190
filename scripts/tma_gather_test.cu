// Standalone probe: TMA tile::gather4 tensor-map encoding, SWIZZLE_{128,64,32}B layouts and
// out-of-bounds zero fill on sm_100a.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// scripts/tma_gather_test.cu -o /tmp/tma_gather_test -lcuda   (run on the GPU box)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void k_gather(const __grid_constant__ CUtensorMap tm, int4 rows, int col, uint16_t *out, int bytes) {
    __shared__ __align__(1024) uint8_t buf[4096];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(buf);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4096; ++i) buf[i] = 0xAB;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4, %5, %6}], [%7];" ::"r"(d),
            "l"(&tm), "r"(col), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w), "r"(b)
            : "memory");
        uint32_t ok = 0;
        for (int spin = 0; spin < 1000000 && !ok; ++spin)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}"
                         : "=r"(ok)
                         : "r"(b));
        out[2047] = ok ? 1 : 0;
        for (int i = 0; i < 2047 && i * 2 < 4096; ++i) out[i] = reinterpret_cast<uint16_t *>(buf)[i];
    }
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no entry point\n"); return 1; }
    const int N = 1000, C = 256;
    std::vector<uint16_t> h((size_t)N * C);
    for (int r = 0; r < N; ++r)
        for (int c = 0; c < C; ++c) h[(size_t)r * C + c] = (uint16_t)(((r & 0x3FF) << 6) ^ (c & 63) ^ ((c >> 6) << 14));
    uint16_t *dF, *dO;
    cudaMalloc(&dF, h.size() * 2);
    cudaMalloc(&dO, 4096 * 2);
    cudaMemcpy(dF, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    struct Mode { CUtensorMapSwizzle sw; int box_cols; const char *name; };
    Mode modes[] = {{CU_TENSOR_MAP_SWIZZLE_128B, 64, "SW128/64cols"}, {CU_TENSOR_MAP_SWIZZLE_64B, 32, "SW64/32cols"},
                    {CU_TENSOR_MAP_SWIZZLE_32B, 16, "SW32/16cols"}, {CU_TENSOR_MAP_SWIZZLE_NONE, 8, "NONE/8cols"}};
    for (auto &m : modes)
        for (int boxh : {1}) {
            CUtensorMap tm;
            cuuint64_t gdim[2] = {(cuuint64_t)C, (cuuint64_t)N};
            cuuint64_t gstride[1] = {(cuuint64_t)C * 2};
            cuuint32_t box[2] = {(cuuint32_t)m.box_cols, (cuuint32_t)boxh};
            cuuint32_t estr[2] = {1, 1};
            CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, dF, gdim, gstride, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, m.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) { printf("%s boxh=%d: encode failed %d\n", m.name, boxh, (int)r); continue; }
            const int rb = m.box_cols * 2;   // bytes per gathered row
            int4 rows = make_int4(5, 900, N + 3, 7);   // third row out of bounds
            const int col = 64;                        // start column (second 64-col chunk)
            cudaMemset(dO, 0, 4096 * 2);
            k_gather<<<1, 32>>>(tm, rows, col, dO, 4 * rb);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("%s boxh=%d: kernel error %s\n", m.name, boxh, cudaGetErrorString(e)); return 2; }
            std::vector<uint16_t> o(4096);
            cudaMemcpy(o.data(), dO, 4096 * 2, cudaMemcpyDeviceToHost);
            // expected: row slot s at s*rb; 16-byte chunk j of the row stored at chunk j ^ f(s)
            int bad = 0, bad_noswz = 0;
            for (int s = 0; s < 4; ++s) {
                int rr = s == 0 ? rows.x : s == 1 ? rows.y : s == 2 ? rows.z : rows.w;
                for (int c = 0; c < m.box_cols; ++c) {
                    uint16_t exp = (rr >= N) ? 0 : h[(size_t)rr * C + col + c];
                    int j = c / 8, e8 = c % 8;
                    int f = m.sw == CU_TENSOR_MAP_SWIZZLE_128B ? (s & 7)
                          : m.sw == CU_TENSOR_MAP_SWIZZLE_64B ? ((s >> 1) & 3)
                          : m.sw == CU_TENSOR_MAP_SWIZZLE_32B ? ((s >> 2) & 1) : 0;
                    int addr = s * rb + ((j ^ f) * 16) + e8 * 2;
                    if (o[addr / 2] != exp) ++bad;
                    if (o[(s * rb + c * 2) / 2] != exp) ++bad_noswz;
                }
            }
            printf("%s boxh=%d: barrier_ok=%d mismatches(swizzle model)=%d mismatches(linear)=%d  first=%04x %04x\n",
                   m.name, boxh, o[2047], bad, bad_noswz, o[0], o[1]);
        }
    return 0;
}
