// spc_dense.cu -- A11: the dense part of the feature computation.  The centre offset of a
// submanifold map is the identity (every output matches itself: the centre column
// is 100% dense) and a K = 1 layer is nothing else, so out = F_in * W_k is a plain dense
// GEMM with no gather at all:
//   warp 0   TMA producer: per (128-row tile, C_in chunk) one cp.async.bulk.tensor 2-D tile
//            load of F_in (box {BK, 128}, written by the TMA unit straight into the
//            UMMA K-major 128B/64B/32B-swizzled layout; rows past the end zero-filled)
//            and one 1-D bulk copy of the pre-tiled weight blob (spc_prepare_weight)
//   warp 1   MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M = 128, N = C_out tile,
//            fp32 accumulator in TMEM (double-buffered across tiles), tcgen05.commit
//   warps 2-5 epilogue: tcgen05.ld -> final dtype + fused residual (K = 1 layers), or an
//            fp32 STORE that initialises the accumulator of a weight-stationary layer
//            (the centre product replaces the zero fill and the centre's pair list)
// Persistent: one CTA per SM, 128-row tiles round-robin; the live row count is read on
// the device (n_dev), so capacity-sized network passes need no host sync.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "spc_common.cuh"
#include "spc_ptx.cuh"
#include "spc_tile.cuh"

namespace spc {

constexpr int DN_THREADS = 192;   // 6 warps: TMA producer, MMA issuer, 4 epilogue warps
constexpr int DN_BM = 128;
constexpr int DN_SMEM_BUDGET = 200 * 1024;
constexpr int DN_MAX_STAGES = 8;

struct DenseParams {
    CUtensorMap tmap_a;        // F_in rows: 2-D {c_in, n_cap}, box {BK, 128}, swizzle = 2*BK bytes
    const char *wblob;         // prepared weights [k_vol][n_ntiles][n_chunks] blobs
    int k;                     // weight offset used (K=1: 0; submanifold centre: (K^3-1)/2)
    int n_chunks, n_ntiles, BK, BN;
    uint32_t kb_a, kb_b;       // bytes of one A / B K-block
    uint32_t a_off, b_off;     // ring offsets of the A / B stages (1024-aligned)
    int stages;
    int64_t n_cap;
    const int64_t *n_dev;
    uint32_t tmem_cols;
    uint32_t idesc;
    // output (store_row interface)
    void *out;
    int64_t ld_out;
    int out_kind;
    int out_dtype;
    const void *residual;
    int64_t ld_res;
    Epi epi;                   // fused BN / ReLU of OUT_FINAL stores (spc_tile.cuh)
    Trace trace;
};

struct DenseSmem {
    uint64_t full[DN_MAX_STAGES], empty[DN_MAX_STAGES], tfull[2], tempty[2];
    uint32_t tmem_holder[4];
};

__global__ void __launch_bounds__(DN_THREADS, 1) k_dense_tc(const __grid_constant__ DenseParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    DenseSmem &ds = *reinterpret_cast<DenseSmem *>(smem);
    const uint32_t sa = ptx::smem_u32(smem + p.a_off), sb = ptx::smem_u32(smem + p.b_off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            ptx::mbar_init(ptx::smem_u32(&ds.full[s]), 1);   // producer's expect_tx arrival
            ptx::mbar_init(ptx::smem_u32(&ds.empty[s]), 1);  // MMA commit
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(ptx::smem_u32(&ds.tfull[a]), 1);
            ptx::mbar_init(ptx::smem_u32(&ds.tempty[a]), 4);
        }
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&p.tmap_a);
        trace_event(p.trace, 0, 0);
    }
    if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(ds.tmem_holder), 2 * p.tmem_cols);
    // barrier init and TMEM allocation overlap the previous kernel's tail (PDL)
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) trace_event(p.trace, 1, 0);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = ds.tmem_holder[0];
    const int64_t n = dev_count(p.n_cap, p.n_dev);
    const int64_t n_tiles = ((n + DN_BM - 1) / DN_BM) * p.n_ntiles;
    constexpr uint32_t MMA_K_BYTES = 32;   // K = 16 bf16 / f16 per tcgen05.mma

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            uint32_t it = 0;
            for (int64_t v = blockIdx.x; v < n_tiles; v += gridDim.x) {
                const int64_t m = v / p.n_ntiles;
                const int nt = (int)(v - m * p.n_ntiles);
                for (int cc = 0; cc < p.n_chunks; ++cc, ++it) {
                    const int s = it % p.stages;
                    ptx::mbar_wait(ptx::smem_u32(&ds.empty[s]), ((it / p.stages) & 1) ^ 1);
                    const uint32_t fb = ptx::smem_u32(&ds.full[s]);
                    ptx::mbar_arrive_expect_tx(fb, p.kb_a + p.kb_b);
                    ptx::tma_load_2d(sa + s * p.kb_a, &p.tmap_a, cc * p.BK, (int)(m * DN_BM), fb);
                    const int64_t blob = ((int64_t)p.k * p.n_ntiles + nt) * p.n_chunks + cc;
                    ptx::bulk_g2s(sb + s * p.kb_b, p.wblob + blob * p.kb_b, p.kb_b, fb);
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (whole warp, elected lane issues) ============
        uint32_t it = 0, ti = 0;
        const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base, 0);
        for (int64_t v = blockIdx.x; v < n_tiles; v += gridDim.x, ++ti) {
            const uint32_t a = ti & 1;
            ptx::mbar_wait(ptx::smem_u32(&ds.tempty[a]), ((ti >> 1) & 1) ^ 1);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tb + a * p.tmem_cols;
            for (int cc = 0; cc < p.n_chunks; ++cc, ++it) {
                const int s = it % p.stages;
                ptx::mbar_wait(ptx::smem_u32(&ds.full[s]), (it / p.stages) & 1);
                ptx::tc_fence_after();
                const uint32_t rb = (uint32_t)p.BK * 2;
                const uint64_t a_d = ptx::umma_desc_kmajor_sw(sa + s * p.kb_a, rb);
                const uint64_t b_d = ptx::umma_desc_kmajor_sw(sb + s * p.kb_b, rb);
                // BK/16 K steps: descriptors advance by 32 bytes (+2 in the address field)
                for (int kk = 0; kk < p.BK / 16; ++kk)
                    ptx::mma_f16_ss_elect(d_tmem, a_d + (kk * MMA_K_BYTES >> 4), b_d + (kk * MMA_K_BYTES >> 4), p.idesc,
                                          (cc | kk) ? 1u : 0u);
                ptx::mma_commit_elect(ptx::smem_u32(&ds.empty[s]));
            }
            ptx::mma_commit_elect(ptx::smem_u32(&ds.tfull[a]));
        }
    } else {
        // ===================== epilogue (thread = TMEM lane = tile row) ===================
        const int q = warp & 3;   // the TMEM lane quadrant this warp may access
        uint32_t ti = 0;
        for (int64_t v = blockIdx.x; v < n_tiles; v += gridDim.x, ++ti) {
            const int64_t m = v / p.n_ntiles;
            const int nt = (int)(v - m * p.n_ntiles);
            const uint32_t a = ti & 1;
            ptx::mbar_wait_sleep(ptx::smem_u32(&ds.tfull[a]), (ti >> 1) & 1);
            ptx::tc_fence_after();
            const int64_t row = m * DN_BM + q * 32 + lane;
            const uint32_t tbase = tmem_base + a * p.tmem_cols + ((uint32_t)(q * 32) << 16);
            for (int col = 0; col < p.BN; col += 32) {
                uint32_t vals[32];
                const int cnt = min(32, p.BN - col);
                if (cnt == 32) ptx::tmem_ld32(tbase + col, vals);
                else ptx::tmem_ld16(tbase + col, vals);
                ptx::tmem_ld_wait();
                if (row < n) {
                    if (p.out_kind == OUT_FINAL && (p.epi.scale || p.epi.shift))
                        epi_affine_u32(p.epi, vals, nt * p.BN + col, cnt);
                    store_row(p, row, nt * p.BN + col, vals, cnt);
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&ds.tempty[a]));
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) trace_event(p.trace, 7, 0);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, 2 * p.tmem_cols);
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

// F_in as a 2-D tensor {c_in (inner), n_rows} with row pitch ld_bytes; box {BK, 128}; the
// swizzle span equals the box row (2*BK bytes), which is the UMMA canonical K-major layout
static spc_status encode_rows_tmap(CUtensorMap *tm, const void *base, int64_t n_rows, int c_in, int64_t ld_bytes,
                                   int BK, int dtype) {
    auto enc = tmap_encoder();
    if (!enc) return fail(SPC_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    const int rb = BK * 2;
    const CUtensorMapSwizzle sw =
        rb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    cuuint64_t gdim[2] = {(cuuint64_t)c_in, (cuuint64_t)(n_rows > 0 ? n_rows : 1)};
    cuuint64_t gstride[1] = {(cuuint64_t)ld_bytes};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)DN_BM};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(tm, dtype == SPC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                     const_cast<void *>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SPC_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return SPC_OK;
}

// out[i] (op)= F_in[i] * W_k for the live rows i < *n_dev of an identity map (K = 1, or a
// submanifold centre).  out_kind: OUT_FINAL (dtype + residual) or OUT_F32_STORE.
spc_status dense_forward(const void *f_in, int64_t ld_in, int in_dtype, int c_in, const void *wblob, int k, int c_out,
                         int BK, int BN, int64_t n_cap, const int64_t *n_dev, void *out, int64_t ld_out, int out_kind,
                         int out_dtype, const void *residual, int64_t ld_res, const Epi &epi, cudaStream_t st) {
    if (n_cap == 0) return SPC_OK;
    DenseParams p;
    memset(&p, 0, sizeof(p));
    spc_status s = encode_rows_tmap(&p.tmap_a, f_in, n_cap, c_in, ld_in * 2, BK, in_dtype);
    if (s != SPC_OK) return s;
    p.wblob = static_cast<const char *>(wblob);
    p.k = k;
    p.BK = BK;
    p.BN = BN;
    p.n_chunks = c_in / BK;
    p.n_ntiles = c_out / BN;
    p.kb_a = (uint32_t)(DN_BM * BK * 2);
    p.kb_b = (uint32_t)(BN * BK * 2);
    p.n_cap = n_cap;
    p.n_dev = n_dev;
    p.tmem_cols = 32;
    while ((int)p.tmem_cols < BN) p.tmem_cols <<= 1;
    p.idesc = ptx::umma_idesc_f16(in_dtype == SPC_BF16, DN_BM, BN);
    p.out = out;
    p.ld_out = ld_out;
    p.out_kind = out_kind;
    p.out_dtype = out_dtype;
    p.residual = residual;
    p.ld_res = ld_res;
    p.epi = epi;
    const size_t hdr = align_up(sizeof(DenseSmem), 1024);
    const size_t per = align_up(p.kb_a, 1024) + align_up(p.kb_b, 1024);
    p.stages = (int)std::min<size_t>(DN_MAX_STAGES, (DN_SMEM_BUDGET - 1024 - hdr) / per);
    if (p.stages < 2) return fail(SPC_ERR_UNSUPPORTED, "dense_forward: tile does not fit shared memory");
    // A stages are 1024-aligned (128B swizzle atoms); kb_a is a multiple of 1024 for BK >= 32
    // and of 512 for BK = 16 (32B swizzle needs 256-byte alignment)
    p.a_off = (uint32_t)hdr;
    p.b_off = (uint32_t)align_up(hdr + (size_t)p.stages * p.kb_a, 1024);
    const size_t smem = 1024 + p.b_off + (size_t)p.stages * p.kb_b;
    static uint64_t configured = 0;   // bit d: attribute set on device d
    const int dev = current_device();
    if (!(configured >> dev & 1)) {
        SPC_CUDA(cudaFuncSetAttribute(k_dense_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, DN_SMEM_BUDGET + 1024));
        configured |= 1ull << dev;
    }
    const int64_t tiles_cap = ((n_cap + DN_BM - 1) / DN_BM) * p.n_ntiles;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles_cap, num_sms()));
    if (option(SPC_OPT_CONV_MAX_CTAS) > 0) grid = (int)std::min<int64_t>(grid, option(SPC_OPT_CONV_MAX_CTAS));
    p.trace = trace_next("k_dense_tc n=" + std::to_string(n_cap) + " c_in=" + std::to_string(c_in) +
                         " c_out=" + std::to_string(c_out) + " k=" + std::to_string(k));
    SPC_CUDA(launch_pdl(k_dense_tc, dim3(grid), dim3(DN_THREADS), smem, st, p));
    SPC_LAUNCH_CHECK("k_dense_tc");
    return SPC_OK;
}

}  // namespace spc
