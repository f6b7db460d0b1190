// spc_wgrad.cu -- SURVEY NEXT-4 training path: the weight gradient of Eq. (2)
// (§2.1; training is beyond the paper's inference scope):
//
//     dW_k[c][o] += sum over the map's pairs (j, i) at offset k of  F_in[j][c] * dF_out[i][o]
//
// a per-offset gather-GEMM whose contraction runs over the PAIRS (M = c_in, N = c_out,
// K = pairs).  Both operands are gathered rows (F_in rows j, dF_out rows i), so a stage
// holds 64 pairs pair-major: row p = one pair's 128 input channels (A) or NP output
// channels (B), 128-byte swizzled rows exactly as the forward gather writes them.  For the
// MMA that is an MN-major operand (the channels, i.e. M resp. N, are contiguous; the pairs,
// i.e. K, step by rows), which tcgen05 reads directly through the transpose bits of the
// instruction descriptor -- no transpose pass, no staging of F_in^T.
//
// Work: sources = the dense (OS) columns of the map (pairs (os_table[i][c], i), sentinel
// rows zero-filled, 128-row chunks with an empty tile mask skipped), its WS lists (pairs
// (j, i)) and, for halved submanifold lists, the mirrored pairs (i, j) at offset
// K^3-1-k.  A work item = (source, range of pairs, 128-channel c_in tile, NP-column
// c_out tile); items are walked round-robin by a persistent grid (counts read on the
// device, so no host sync).  Each item accumulates in TMEM and is reduced into the fp32
// dW with red.global.add.v4.f32 (items of one offset overlap only through those adds).
//
//   warps 0-7  gather (one stage each, round-robin): cp.async 16-byte row segments (zero-fill for sentinels, pairs past
//              the end and channels past c_in / c_out), completion on the stage mbarrier
//   warps 8-11 epilogue: tcgen05.ld (thread = c_in row) -> red.global.add.v4.f32 into dW
//   warp 12    TMEM allocation + MMA issue (tcgen05.mma kind::f16, M = 128, N = NP,
//              A and B MN-major SWIZZLE_128B), accumulators double-buffered across items
#include <cuda_runtime.h>

#include "spc_common.cuh"
#include "spc_ptx.cuh"
#include "spc_tile.cuh"

namespace spc {

constexpr int WG_GATHER = 8;              // producer warps
constexpr int WG_MMA_WARP = WG_GATHER + 4;
constexpr int WG_THREADS = 32 * (WG_GATHER + 5);
constexpr int WG_PAIRS = 64;                 // pairs per stage (4 K=16 MMAs)
constexpr int WG_M = 128;                    // c_in channels per item (TMEM lanes)
constexpr int WG_ATOM = WG_PAIRS * 128;      // bytes of one 64-channel column of a stage
constexpr int WG_MAX_SRC = 2 * SPC_MAX_KVOL + 1;
constexpr int WG_MAX_STAGES = 12;
constexpr int WG_SMEM_BUDGET = 210 * 1024;

struct WgradParams {
    const char *f_in;
    int64_t ld_in_bytes;
    int c_in;
    const char *d_out;
    int64_t ld_dout_bytes;
    int c_out;
    float *dw;                      // [k_vol][c_in][c_out] fp32, accumulated
    const int32_t *os;
    int k_dense;
    const uint32_t *tile_mask;
    int tile_words;
    const int2 *pairs;
    int64_t list_stride;
    const int32_t *counts;
    int64_t n_out_cap;
    const int64_t *n_out_dev;
    int range;                      // pairs per work item (multiple of WG_PAIRS)
    int n_mt, n_nt, NP;
    uint32_t a_bytes, b_bytes;      // per stage
    int stages;
    uint32_t tmem_cols;
    uint32_t idesc;
    int n_src;
    int16_t src_k[WG_MAX_SRC];      // weight offset the source contributes to
    int16_t src_idx[WG_MAX_SRC];    // dense column / list index
    int8_t src_kind[WG_MAX_SRC];    // 0 dense column, 1 list, 2 mirrored list
    Trace trace;
};

struct WgradSmem {
    uint64_t full[WG_MAX_STAGES], empty[WG_MAX_STAGES], tfull[2], tempty[2];
    uint32_t tmem_holder[4];
    int64_t item_start[WG_MAX_SRC + 1];   // prefix over sources of their work items
    int64_t src_pairs[WG_MAX_SRC];
};

struct WItem {
    int src, mt, nt;
    int64_t p0, p1;
};

__device__ __forceinline__ WItem decode_item(const WgradParams &p, const WgradSmem &ws, int64_t v) {
    int s = 0;
    while (ws.item_start[s + 1] <= v) ++s;
    int64_t r = v - ws.item_start[s];
    WItem it;
    it.src = s;
    it.nt = (int)(r % p.n_nt);
    r /= p.n_nt;
    it.mt = (int)(r % p.n_mt);
    r /= p.n_mt;
    it.p0 = r * p.range;
    it.p1 = imin64(ws.src_pairs[s], it.p0 + p.range);
    return it;
}

// a stage of a dense-column source is skipped when its 128-output tile has no match at
// that column (tile masks of the OS table); list stages always run
__device__ __forceinline__ bool stage_active(const WgradParams &p, const WItem &it, int64_t q0) {
    if (p.src_kind[it.src] != 0) return true;
    const int c = p.src_idx[it.src];
    const int64_t tile = q0 >> 7;
    return (__ldg(p.tile_mask + tile * p.tile_words + (c >> 5)) >> (c & 31)) & 1u;
}

__device__ __forceinline__ int active_stages(const WgradParams &p, const WItem &it) {
    int n = 0;
    for (int64_t q0 = it.p0; q0 < it.p1; q0 += WG_PAIRS) n += stage_active(p, it, q0) ? 1 : 0;
    return n;
}

// MN-major SWIZZLE_128B descriptor: 64-element (128-byte) MN atoms LBO apart, 8-row K
// groups SBO = 1024 bytes apart (CUTLASS canonical ((8,n),(8,k)):((1,LBO),(8,SBO)) in 16-B units)
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t addr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;   // SWIZZLE_128B
    return d;
}

__global__ void __launch_bounds__(WG_THREADS, 1) k_wgrad_tc(const __grid_constant__ WgradParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    WgradSmem &ws = *reinterpret_cast<WgradSmem *>(smem);
    uint8_t *ring = smem + ((sizeof(WgradSmem) + 1023) & ~size_t(1023));
    const uint32_t ring_u32 = ptx::smem_u32(ring);
    const uint32_t stage_bytes = p.a_bytes + p.b_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            ptx::mbar_init(ptx::smem_u32(&ws.full[s]), 32);    // one noinc arrival per lane of the filling warp
            ptx::mbar_init(ptx::smem_u32(&ws.empty[s]), 1);    // MMA commit
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(ptx::smem_u32(&ws.tfull[a]), 1);
            ptx::mbar_init(ptx::smem_u32(&ws.tempty[a]), 4);
        }
        ptx::fence_mbar_init();
        trace_event(p.trace, 0, 0);
    }
    if (warp == WG_MMA_WARP) ptx::tmem_alloc(ptx::smem_u32(ws.tmem_holder), 2 * p.tmem_cols);
    pdl_wait();   // the map, its counts, F_in and dF_out come from preceding kernels
    pdl_trigger();
    if (threadIdx.x == 0) {
        const int64_t n_out = dev_count(p.n_out_cap, p.n_out_dev);
        int64_t acc = 0;
        for (int s = 0; s < p.n_src; ++s) {
            const int64_t np = p.src_kind[s] == 0 ? n_out : (int64_t)p.counts[SPC_MAX_KVOL + p.src_idx[s]];
            ws.src_pairs[s] = np;
            ws.item_start[s] = acc;
            acc += (np + p.range - 1) / p.range * p.n_mt * p.n_nt;
        }
        ws.item_start[p.n_src] = acc;
        trace_event(p.trace, 1, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = ws.tmem_holder[0];
    const int64_t n_items = ws.item_start[p.n_src];

    if (warp < WG_GATHER) {
        // ===================== gather (WG_GATHER warps, one stage each, round-robin) =====
        // channels past c_in / c_out are the same for every stage when the launch has one
        // c_in / c_out tile (and the valid chunk count is a power of two): zero them in the
        // whole ring once instead of zero-filling per stage
        const bool pre_a = p.n_mt == 1 && p.c_in < WG_M && ((p.c_in / 8) & (p.c_in / 8 - 1)) == 0;
        const bool pre_b = p.n_nt == 1 && p.c_out < p.NP && ((p.c_out / 8) & (p.c_out / 8 - 1)) == 0;
        if (pre_a || pre_b) {
            for (int s = 0; s < p.stages; ++s) {
                uint4 *a = reinterpret_cast<uint4 *>(ring + s * stage_bytes);
                for (int e = threadIdx.x; e < (int)(stage_bytes / 16); e += 32 * WG_GATHER) {
                    const bool in_a = e < (int)(p.a_bytes / 16);
                    const int off = in_a ? e : e - (int)(p.a_bytes / 16);
                    const int col = off / (WG_ATOM / 16), r = (off % (WG_ATOM / 16)) / 8, c16 = (off % 8) ^ (r & 7);
                    const int ch = col * 8 + c16;   // 16-byte chunk (8 channels) of the row
                    if ((in_a && pre_a && ch * 8 >= p.c_in) || (!in_a && pre_b && ch * 8 >= p.c_out))
                        a[e] = make_uint4(0, 0, 0, 0);
                }
            }
            ptx::fence_proxy_async();
            asm volatile("bar.sync 2, %0;" ::"n"(32 * WG_GATHER) : "memory");   // every producer's zeros before any arrival
        }
        const int a_sh = __ffs(pre_a ? p.c_in / 8 : 16) - 1;     // log2(chunks issued per A row)
        const int b_sh = __ffs(pre_b ? p.c_out / 8 : p.NP / 8) - 1;
        // cursor over the (item, active stage) sequence every role walks; warp w fills the
        // stages it = w, w + 4, ... and prefetches its next stage's indices before issuing
        struct Cur {
            int64_t v, q0;
            WItem w;
        };
        auto settle = [&](Cur &c) {   // move to the first active stage at or after c.q0
            while (c.v < n_items) {
                while (c.q0 < c.w.p1 && !stage_active(p, c.w, c.q0)) c.q0 += WG_PAIRS;
                if (c.q0 < c.w.p1) return;
                c.v += gridDim.x;
                if (c.v < n_items) {
                    c.w = decode_item(p, ws, c.v);
                    c.q0 = c.w.p0;
                }
            }
        };
        auto step = [&](Cur &c, int n) {
            for (int k = 0; k < n && c.v < n_items; ++k) {
                c.q0 += WG_PAIRS;
                settle(c);
            }
        };
        // (j, i) of pairs q0 + lane and q0 + 32 + lane of the cursor's stage
        auto fetch = [&](const Cur &c, int (&j)[2], int (&i)[2]) {
            const int kind = p.src_kind[c.w.src], idx = p.src_idx[c.w.src];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                j[h] = -1;
                i[h] = -1;
                const int64_t q = c.q0 + 32 * h + lane;
                if (q < c.w.p1) {
                    if (kind == 0) {
                        j[h] = __ldg(p.os + q * p.k_dense + idx);
                        i[h] = (int)q;
                    } else {
                        const int2 pr = __ldg(p.pairs + idx * p.list_stride + q);
                        j[h] = kind == 1 ? pr.x : pr.y;
                        i[h] = kind == 1 ? pr.y : pr.x;
                    }
                }
            }
        };
        Cur cur;
        cur.v = blockIdx.x;
        cur.q0 = 0;
        if (cur.v < n_items) {
            cur.w = decode_item(p, ws, cur.v);
            cur.q0 = cur.w.p0;
        }
        settle(cur);
        // a warp may run at most one ring phase ahead of its slot's previous user: with W
        // producers filling stages round-robin that needs W <= stages (mbarrier parity waits
        // cannot tell two phases apart)
        const int WA = min(WG_GATHER, p.stages);
        if (warp >= WA) cur.v = n_items;   // idle producer
        step(cur, warp);
        uint32_t it = warp;
        // indices of this warp's next two stages are in flight while it fills the current one
        // (the pair lists / OS columns live in L2 or HBM: one stage of lead hid too little)
        Cur nxt = cur;
        step(nxt, WA);
        int jn[2], in_[2], jn2[2], in2[2];
        if (cur.v < n_items) fetch(cur, jn, in_);
        if (nxt.v < n_items) fetch(nxt, jn2, in2);
        while (cur.v < n_items) {
            const Cur c = cur;
            const int j[2] = {jn[0], jn[1]}, i[2] = {in_[0], in_[1]};
            cur = nxt;
            jn[0] = jn2[0], jn[1] = jn2[1], in_[0] = in2[0], in_[1] = in2[1];
            step(nxt, WA);
            if (nxt.v < n_items) fetch(nxt, jn2, in2);
            const int s = it % p.stages;
            ptx::mbar_wait(ptx::smem_u32(&ws.empty[s]), ((it / p.stages) & 1) ^ 1);
            const uint32_t sA = ring_u32 + s * stage_bytes, sB = sA + p.a_bytes;
            const int m0 = c.w.mt * WG_M, n0 = c.w.nt * p.NP;
            // A: 64 pairs x 2^a_sh chunks (channels m0.. of F_in row j), pair-major across lanes
            for (int e = lane; e < (64 << a_sh); e += 32) {
                const int pp = e >> a_sh, ch = e & ((1 << a_sh) - 1);
                const int lo = __shfl_sync(0xffffffffu, j[0], pp & 31), hi = __shfl_sync(0xffffffffu, j[1], pp & 31);
                const int jj = pp < 32 ? lo : hi;
                const int ci = m0 + ch * 8;
                const bool ok = jj >= 0 && ci < p.c_in;
                const uint32_t dst = sA + (ch >> 3) * WG_ATOM + pp * 128 + (((ch & 7) ^ (pp & 7)) << 4);
                ptx::cp_async_16(dst, ok ? p.f_in + (int64_t)jj * p.ld_in_bytes + ci * 2 : p.f_in, ok ? 16u : 0u);
            }
            // B: 64 pairs x 2^b_sh chunks (channels n0.. of dF_out row i); a sentinel pair
            // contributes nothing, so its B row is zero-filled too (no load)
            for (int e = lane; e < (64 << b_sh); e += 32) {
                const int pp = e >> b_sh, ch = e & ((1 << b_sh) - 1);
                const int jl = __shfl_sync(0xffffffffu, j[0], pp & 31), jh = __shfl_sync(0xffffffffu, j[1], pp & 31);
                const int il = __shfl_sync(0xffffffffu, i[0], pp & 31), ih = __shfl_sync(0xffffffffu, i[1], pp & 31);
                const int jj = pp < 32 ? jl : jh, ii = pp < 32 ? il : ih;
                const int co = n0 + ch * 8;
                const bool ok = jj >= 0 && ii >= 0 && co < p.c_out;
                const uint32_t dst = sB + (ch >> 3) * WG_ATOM + pp * 128 + (((ch & 7) ^ (pp & 7)) << 4);
                ptx::cp_async_16(dst, ok ? p.d_out + (int64_t)ii * p.ld_dout_bytes + co * 2 : p.d_out,
                                 ok ? 16u : 0u);
            }
            ptx::fence_proxy_async();
            ptx::cp_async_mbar_arrive(ptx::smem_u32(&ws.full[s]));
            it += WA;
        }
        ptx::cp_async_wait<0>();
    } else if (warp == WG_MMA_WARP) {
        // ===================== MMA issuer =====================
        uint32_t it = 0, ti = 0;
        const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base, 0);
        for (int64_t v = blockIdx.x; v < n_items; v += gridDim.x) {
            const WItem w = decode_item(p, ws, v);
            if (active_stages(p, w) == 0) continue;
            const uint32_t a = ti & 1;
            ptx::mbar_wait(ptx::smem_u32(&ws.tempty[a]), ((ti >> 1) & 1) ^ 1);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tb + a * p.tmem_cols;
            bool first = true;
            for (int64_t q0 = w.p0; q0 < w.p1; q0 += WG_PAIRS) {
                if (!stage_active(p, w, q0)) continue;
                const int s = it % p.stages;
                ptx::mbar_wait(ptx::smem_u32(&ws.full[s]), (it / p.stages) & 1);
                ptx::tc_fence_after();
                const uint32_t sA = ring_u32 + s * stage_bytes, sB = sA + p.a_bytes;
                const uint64_t ad = desc_mn_sw128(sA, WG_ATOM), bd = desc_mn_sw128(sB, WG_ATOM);
                // K = 16 pairs per MMA = two 8-row groups: +2048 bytes (+128 in the address field)
#pragma unroll
                for (int kk = 0; kk < WG_PAIRS / 16; ++kk)
                    ptx::mma_f16_ss_elect(d_tmem, ad + 128 * kk, bd + 128 * kk, p.idesc, (first && kk == 0) ? 0u : 1u);
                first = false;
                ptx::mma_commit_elect(ptx::smem_u32(&ws.empty[s]));
                ++it;
            }
            ptx::mma_commit_elect(ptx::smem_u32(&ws.tfull[a]));
            ++ti;
        }
    } else {
        // ===================== epilogue (thread = TMEM lane = c_in row) ===================
        const int q = warp & 3;
        uint32_t ti = 0;
        for (int64_t v = blockIdx.x; v < n_items; v += gridDim.x) {
            const WItem w = decode_item(p, ws, v);
            if (active_stages(p, w) == 0) continue;
            const uint32_t a = ti & 1;
            ptx::mbar_wait_sleep(ptx::smem_u32(&ws.tfull[a]), (ti >> 1) & 1);
            ptx::tc_fence_after();
            const int ci = w.mt * WG_M + q * 32 + lane;
            const int n0 = w.nt * p.NP;
            float *row = p.dw + ((int64_t)p.src_k[w.src] * p.c_in + ci) * p.c_out;
            const uint32_t tbase = tmem_base + a * p.tmem_cols + ((uint32_t)(q * 32) << 16);
            for (int col = 0; col < p.NP; col += 32) {
                uint32_t vals[32];
                ptx::tmem_ld32(tbase + col, vals);
                ptx::tmem_ld_wait();
                if (ci < p.c_in) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int co = n0 + col + 4 * e;
                        if (co < p.c_out)
                            ptx::red_add_v4(row + co, to_f(vals[4 * e]), to_f(vals[4 * e + 1]), to_f(vals[4 * e + 2]),
                                            to_f(vals[4 * e + 3]));
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&ws.tempty[a]));
            ++ti;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) trace_event(p.trace, 7, 0);
    if (warp == WG_MMA_WARP) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, 2 * p.tmem_cols);
    }
}

// fp32 path (FFMA): one 32x32 (c_in x c_out) tile of one source's pair range per block;
// pairs staged 32 at a time in shared memory, partial sums added with atomics
constexpr int WS_TP = 32;
__global__ void __launch_bounds__(256) k_wgrad_simt(const __grid_constant__ WgradParams p) {
    __shared__ float sf[WS_TP][WS_TP + 1], sg[WS_TP][WS_TP + 1];
    __shared__ int64_t start[WG_MAX_SRC + 1], npairs[WG_MAX_SRC];
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) {
        const int64_t n_out = dev_count(p.n_out_cap, p.n_out_dev);
        int64_t acc = 0;
        for (int s = 0; s < p.n_src; ++s) {
            const int64_t np = p.src_kind[s] == 0 ? n_out : (int64_t)p.counts[SPC_MAX_KVOL + p.src_idx[s]];
            npairs[s] = np;
            start[s] = acc;
            acc += (np + p.range - 1) / p.range * p.n_mt * p.n_nt;
        }
        start[p.n_src] = acc;
    }
    __syncthreads();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // ty: 8 rows of 4 c_in each
    for (int64_t v = blockIdx.x; v < start[p.n_src]; v += gridDim.x) {
        int s = 0;
        while (start[s + 1] <= v) ++s;
        int64_t r = v - start[s];
        const int nt = (int)(r % p.n_nt);
        r /= p.n_nt;
        const int mt = (int)(r % p.n_mt);
        const int64_t p0 = (r / p.n_mt) * p.range, p1 = imin64(npairs[s], p0 + p.range);
        const int kind = p.src_kind[s], idx = p.src_idx[s];
        const int ci0 = mt * WS_TP, co0 = nt * WS_TP;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int64_t q0 = p0; q0 < p1; q0 += WS_TP) {
            // stage 32 pairs: row t = pair q0 + t; F_in[j][ci0 + 0..31] and dF_out[i][co0 + 0..31]
            for (int e = threadIdx.x; e < WS_TP * WS_TP; e += 256) {
                const int t = e >> 5, c = e & 31;
                const int64_t q = q0 + t;
                int j = -1, i = -1;
                if (q < p1) {
                    if (kind == 0) {
                        j = p.os[q * p.k_dense + idx];
                        i = (int)q;
                    } else {
                        const int2 pr = p.pairs[idx * p.list_stride + q];
                        j = kind == 1 ? pr.x : pr.y;
                        i = kind == 1 ? pr.y : pr.x;
                    }
                }
                const bool ok = j >= 0;
                sf[t][c] = ok && ci0 + c < p.c_in
                               ? reinterpret_cast<const float *>(p.f_in + (int64_t)j * p.ld_in_bytes)[ci0 + c]
                               : 0.f;
                sg[t][c] = ok && co0 + c < p.c_out
                               ? reinterpret_cast<const float *>(p.d_out + (int64_t)i * p.ld_dout_bytes)[co0 + c]
                               : 0.f;
            }
            __syncthreads();
#pragma unroll 8
            for (int t = 0; t < WS_TP; ++t) {
                const float g = sg[t][tx];
#pragma unroll
                for (int m = 0; m < 4; ++m) acc[m] = fmaf(sf[t][ty * 4 + m], g, acc[m]);
            }
            __syncthreads();
        }
        for (int m = 0; m < 4; ++m) {
            const int ci = ci0 + ty * 4 + m, co = co0 + tx;
            if (ci < p.c_in && co < p.c_out) atomicAdd(p.dw + ((int64_t)p.src_k[s] * p.c_in + ci) * p.c_out + co, acc[m]);
        }
    }
}

}  // namespace spc

using namespace spc;

extern "C" spc_status spc_conv_wgrad(const spc_kmap *km, const void *f_in, int64_t ld_in, int32_t in_dtype,
                                     int32_t c_in, const void *d_out, int64_t ld_dout, int32_t c_out, float *d_weight,
                                     void *stream) {
    SPC_CHECK_ARG(km && d_weight, "null pointer");
    SPC_CHECK_ARG(in_dtype >= SPC_F32 && in_dtype <= SPC_BF16, "bad dtype");
    SPC_CHECK_ARG(c_in > 0 && c_out > 0 && ld_in >= c_in && ld_dout >= c_out, "bad channel counts / leading dims");
    SPC_CHECK_ARG((f_in || km->n_in == 0) && (d_out || km->n_out == 0), "null f_in / d_out");
    const size_t es = in_dtype == SPC_F32 ? 4 : 2;
    SPC_CHECK_ARG(((uintptr_t)f_in % 16) == 0 && (ld_in * es) % 16 == 0, "f_in rows must be 16-byte aligned");
    SPC_CHECK_ARG(((uintptr_t)d_out % 16) == 0 && (ld_dout * es) % 16 == 0, "d_out rows must be 16-byte aligned");
    SPC_CHECK_ARG(((uintptr_t)d_weight % 16) == 0, "d_weight must be 16-byte aligned");
    if (km->key_bits != 64 && km->key_bits != 32) return fail(SPC_ERR_INVALID_ARG, "not a built kernel map");
    cudaStream_t st = as_stream(stream);
    if (km->n_out == 0) return SPC_OK;

    WgradParams p;
    memset(&p, 0, sizeof(p));
    p.f_in = static_cast<const char *>(f_in);
    p.ld_in_bytes = ld_in * (int64_t)es;
    p.c_in = c_in;
    p.d_out = static_cast<const char *>(d_out);
    p.ld_dout_bytes = ld_dout * (int64_t)es;
    p.c_out = c_out;
    p.dw = d_weight;
    p.os = km->os_table;
    p.k_dense = km->k_dense;
    p.tile_mask = km->tile_mask_dev;
    p.tile_words = km->tile_words;
    p.pairs = reinterpret_cast<const int2 *>(km->ws_pairs);
    p.list_stride = km->n_out;
    p.counts = km->counts_dev;
    p.n_out_cap = km->n_out;
    p.n_out_dev = km->n_out_dev;
    int ns = 0;
    for (int c = 0; c < km->k_dense; ++c, ++ns) {
        p.src_kind[ns] = 0;
        p.src_idx[ns] = (int16_t)c;
        p.src_k[ns] = km->dense_k[c];
    }
    for (int l = 0; l < km->n_lists; ++l) {
        p.src_kind[ns] = 1;
        p.src_idx[ns] = (int16_t)l;
        p.src_k[ns++] = km->list_k[l];
        if (km->list_mirror[l]) {
            p.src_kind[ns] = 2;
            p.src_idx[ns] = (int16_t)l;
            p.src_k[ns++] = (int16_t)(km->k_vol - 1 - km->list_k[l]);
        }
    }
    p.n_src = ns;
    if (ns == 0) return SPC_OK;
    const int sms = num_sms();
    p.trace = trace_next("k_wgrad n_out=" + std::to_string(km->n_out) + " c_in=" + std::to_string(c_in) +
                         " c_out=" + std::to_string(c_out));

    if (in_dtype == SPC_F32) {
        p.n_mt = (c_in + WS_TP - 1) / WS_TP;
        p.n_nt = (c_out + WS_TP - 1) / WS_TP;
        const int64_t est = (int64_t)ns * km->n_out * p.n_mt * p.n_nt;
        p.range = (int)std::max<int64_t>(WS_TP * 8, std::min<int64_t>(8192, est / (8 * sms) / WS_TP * WS_TP));
        SPC_CUDA(launch_pdl(k_wgrad_simt, dim3((unsigned)(8 * sms)), dim3(256), 0, st, p));
        SPC_LAUNCH_CHECK("k_wgrad_simt");
        return SPC_OK;
    }
    if (c_in % 16 || c_out % 16)
        return fail(SPC_ERR_UNSUPPORTED, "spc_conv_wgrad: f16/bf16 needs c_in and c_out multiples of 16");
    p.NP = c_out <= 64 ? 64 : c_out <= 128 ? 128 : 256;   // power-of-two 16-byte chunks per B row
    p.n_nt = (c_out + p.NP - 1) / p.NP;
    p.n_mt = (c_in + WG_M - 1) / WG_M;
    p.a_bytes = 2 * WG_ATOM;
    p.b_bytes = (uint32_t)(p.NP / 64) * WG_ATOM;
    p.tmem_cols = 32;
    while ((int)p.tmem_cols < p.NP) p.tmem_cols <<= 1;
    // instruction descriptor: f32 accumulate, A and B MN-major (transpose bits 15 / 16)
    p.idesc = ptx::umma_idesc_f16(in_dtype == SPC_BF16, WG_M, p.NP) | (1u << 15) | (1u << 16);
    // ~4 items per SM over the capacity's pairs (the live counts are smaller or equal)
    const int64_t est = (int64_t)ns * km->n_out * p.n_mt * p.n_nt;
    const int64_t ipsm = std::max<int64_t>(1, option(SPC_OPT_WGRAD_ITEMS_PER_SM));
    p.range = (int)std::max<int64_t>(4 * WG_PAIRS,
                                     std::min<int64_t>(64 * WG_PAIRS, est / (ipsm * sms) / WG_PAIRS * WG_PAIRS));
    const size_t hdr = align_up(sizeof(WgradSmem), 1024);
    const size_t per = p.a_bytes + p.b_bytes;
    p.stages = (int)std::min<size_t>(WG_MAX_STAGES, (WG_SMEM_BUDGET - hdr) / per);
    if (p.stages < 2) return fail(SPC_ERR_UNSUPPORTED, "spc_conv_wgrad: stage does not fit shared memory");
    const size_t smem = 1024 + hdr + (size_t)p.stages * per;
    static uint64_t configured = 0;
    const int dev = current_device();
    if (!(configured >> dev & 1)) {
        SPC_CUDA(cudaFuncSetAttribute(k_wgrad_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, WG_SMEM_BUDGET + 2048));
        configured |= 1ull << dev;
    }
    SPC_CUDA(launch_pdl(k_wgrad_tc, dim3((unsigned)sms), dim3(WG_THREADS), smem, st, p));
    SPC_LAUNCH_CHECK("k_wgrad_tc");
    return SPC_OK;
}
