// spc_conv.cu -- A9-A12 feature computation (Eq. 2) with the output-stationary
// and weight-stationary dataflows and the hybrid split.
//
// f16/bf16 path: one persistent, warp-specialised tcgen05 kernel (k_conv_tc), launched
// once for the OS part and once for the WS part of a map:
//   warps 0-3  gather producers: one thread per tile row, cp.async 16-byte row segments
//              (src-size 0 zero-fill for sentinel rows) into the UMMA K-major canonical
//              layout, then fence.proxy.async + mbarrier arrive
//   warp 8     weight producer: one 1-D bulk copy (TMA engine) per stage of the
//              pre-tiled weight blob W_k[c-chunk] (spc_prepare_weight)
//   warp 9     MMA issuer: tcgen05.mma kind::f16, M=128, N=C_out tile, K=16, fp32
//              accumulator in TMEM (double-buffered across tiles), tcgen05.commit
//   warps 4-7  epilogue: tcgen05.ld -> OS: plain stores (final dtype, fused residual, or
//              fp32 accumulator); WS: red.global.add.v4.f32 scatter (P:132 atomics)
// A tile of the OS part is 128 outputs x all dense offsets whose (tile, offset) chunk is
// non-empty (tile mask from the map build); a tile of the WS part is 128 pairs of one
// offset list (plus, for halved submanifold maps, the mirrored product).
//
// f32 path: FFMA kernel with the same tiling semantics (1e-5 accuracy bar; 1xTF32 cannot
// meet it, reading A19).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "spc_common.cuh"
#include "spc_ptx.cuh"
#include "spc_tile.cuh"

namespace spc {

constexpr int TC_THREADS = 480;   // 15 warps: 8 gather, 4 epilogue, MMA, weight loader, scheduler
constexpr int N_GATHER = 8;        // gather warps (two per SM sub-partition)
constexpr int TC_BM = 128;
constexpr int TC_SMEM_BUDGET = 225 * 1024;
constexpr int WS_CTR_SLOTS = 2048;                // ws counters (int32) after the accumulator
constexpr int CTR_EXIT = WS_CTR_SLOTS - 2, CTR_FETCH = WS_CTR_SLOTS - 1;   // split tiles use [0, 1024)
constexpr int SPLIT_MAX_TILES = 512;              // weighted split: tiles per launch (x n_ntiles <= 2)


struct ConvParams {
    int mode;   // 0 = OS part, 1 = WS part
    // map
    const int32_t *os;
    const int32_t *os_rows;   // OS density order: table row -> output row (NULL: identity)
    const int32_t *tile_order;   // OS density order: [2][tiles128] heaviest-first tile orders (or NULL)
    int64_t tiles128_cap;
    int k_dense;
    const uint32_t *tile_mask;
    int tile_words;
    const int2 *pairs;
    int64_t list_stride;
    const int32_t *counts;   // [2*SPC_MAX_KVOL]
    int n_lists;
    int skip_list;        // WS: a list computed elsewhere (the submanifold centre by the dense kernel), or -1
    int k_vol;
    int64_t n_out_cap;
    const int64_t *n_out_dev;
    // operands
    const char *f_in;
    int64_t ld_in_bytes;
    const char *wblob;
    int n_chunks, n_ntiles, BK, BN;
    uint32_t kb_b;        // bytes of one B K-block (BN x BK weight slice)
    // pipeline ring carved per tile height: ring[0] for BM-row tiles, ring[1] for 128-row
    // tiles of a BM=256 kernel (half-height A slices, so more slices per stage)
    struct Ring {
        uint32_t kb_a;     // bytes of one A K-block (tile rows x BK)
        uint32_t a_bytes, b_bytes;   // per stage
        int nkb;           // K-blocks (slices) per stage
        int stages;
    } ring[2];
    uint32_t hdr_off;     // byte offset of ConvSmem + index blocks (after the ring)
    uint32_t red_off;     // byte offset of the WS bulk-reduction staging rows (0: red.global.add)
    int bm;               // max rows per tile (template BM): 128 or 256 (two M=128 MMAs sharing the weight tile)
    int split_ok;         // OS part may split a tile's offsets over CTAs (needs acc + tile_ctr)
    int force_tr;         // experiments: 128/256 forces the tile rows (0 = device heuristic)
    int split_min_unit;   // weighted split: minimum offsets per part
    int claim_ahead;      // dynamic claims: tile ti is claimed once the gather warps began tile ti - claim_ahead
    int split_tiles_per_sm2;   // weighted split when 2 * tiles <= this (default: SM count)
    int num_sms;
    float *acc;           // fp32 split-K accumulator (all-zero on entry, left all-zero)
    int64_t ld_acc;
    int *tile_ctr;        // ws counters (zero on entry, left zero): [0, 1024) split-tile arrivals,
                          // [CTR_EXIT] CTAs exited, [CTR_FETCH] dynamic tile fetch
    int blk_slots;        // gather-index blocks in flight (2, or 1 when a block is large: K=5 OS)
    int maps_ready;       // map + weights complete before the previous kernel started (PDL early start)
    int cg;               // 2: CTA pairs (cta_group::2, M = 256 per MMA, each CTA holds half of every
                          //    weight tile and 128 of the pair tile's 256 rows); 1: single CTAs
    uint32_t tmem_cols;   // per 128-row accumulator (power of two >= 32)
    int tbufs;            // accumulator buffers per CTA: 2 (epilogue overlaps the next tile's MMAs)
                          // or 1 (256-row tiles of N = 256: 2 x 256 columns fill TMEM)
    uint32_t idesc;
    // output
    void *out;
    int64_t ld_out;       // elements
    int out_kind;
    int out_dtype;        // for OUT_FINAL
    const void *residual;
    int64_t ld_res;
    Epi epi;              // fused BN (folded scale / shift) + ReLU of OUT_FINAL stores
    int16_t dense_k[SPC_MAX_KVOL];
    int16_t list_k[SPC_MAX_KVOL];
    int8_t list_mirror[SPC_MAX_KVOL];
    Trace trace;          // device event trace (spc_set_trace), buf NULL = off
};

struct TileInfo {
    int64_t row0;   // first output (OS) or first pair (WS)
    int rows;
    int nt;         // C_out tile
    int list, dir, k;   // OS: list = split part
    int nsplit, ctr;    // OS: parts of this tile (split-K) and its arrival counter slot
    uint32_t mask[4];
};

// virtual tile v -> TileInfo (scheduler warp).  tr = rows per tile, chosen on the device
// from the live counts; OS: sp_pre/sp_cnt (weighted split, or NULL) give each tile's parts.
__device__ __forceinline__ void decode_tile(const ConvParams &p, int64_t v, const int *list_prefix, int64_t n_out,
                                            int tr, const int *sp_pre, const uint16_t *sp_cnt, int n_sp, TileInfo &t) {
    t.nt = (int)(v % p.n_ntiles);
    const int64_t tv = v / p.n_ntiles;
    if (p.mode == 0) {
        int64_t ti = tv;
        t.list = 0;
        t.nsplit = 1;
        if (sp_pre) {   // weighted split: tile = last prefix <= tv
            int lo = 0, hi = n_sp - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (sp_pre[mid] <= tv) lo = mid;
                else hi = mid - 1;
            }
            ti = lo;
            t.list = (int)(tv - sp_pre[lo]);
            t.nsplit = sp_cnt[lo];
        }
        t.ctr = (int)(ti * p.n_ntiles + t.nt);
        int64_t rt = ti;
        if (p.tile_order) rt = p.tile_order[(tr == 256 ? p.tiles128_cap : 0) + rt];   // heaviest first
        t.row0 = rt * tr;
        t.rows = (int)imin64(tr, n_out - t.row0);
        t.dir = 0;
        t.k = -1;
    } else {
        int l = 0;
        while (l + 1 < p.n_lists && list_prefix[l + 1] <= tv) ++l;
        const int local = (int)(tv - list_prefix[l]);
        const int cnt = p.counts[SPC_MAX_KVOL + l];
        const int per = (cnt + tr - 1) / tr;
        t.list = l;
        t.dir = local / per;
        const int tl = local - t.dir * per;
        t.row0 = (int64_t)tl * tr;
        t.rows = min(tr, cnt - tl * tr);
        t.k = t.dir ? p.k_vol - 1 - p.list_k[l] : p.list_k[l];
        t.mask[0] = 1u;
        t.mask[1] = t.mask[2] = t.mask[3] = 0u;
    }
}

// OS: the tile's active offset columns (kernel-map tile mask words of its 128-row tiles)
__device__ __forceinline__ void decode_tile_mask(const ConvParams &p, TileInfo &t) {
    bool any = false;
    const int64_t mt0 = t.row0 / 128, mt1 = (t.row0 + t.rows - 1) / 128;   // kernel-map mask tiles
    for (int w = 0; w < 4; ++w) {
        uint32_t m = 0;
        if (w < p.tile_words)
            for (int64_t mt = mt0; mt <= mt1; ++mt) m |= p.tile_mask[mt * p.tile_words + w];
        t.mask[w] = m;
        any |= t.mask[w] != 0;
    }
    if (!any) t.mask[0] = 1u;   // keep one (all-sentinel) step so the tile is written
}

__device__ __forceinline__ uint32_t ptx_lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ int next_bit(const uint32_t (&m)[4], int from) {
    if (from >= 128) return -1;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        if (w < (from >> 5)) continue;
        uint32_t word = m[w];
        if (w == (from >> 5)) word &= ~0u << (from & 31);
        if (word) return w * 32 + __ffs(word) - 1;
    }
    return -1;
}

// ---- shared-memory records produced by the scheduler warp ------------------------------
constexpr int TREC_SLOTS = 4;      // tile records in flight
constexpr int BLK_SLOTS = 2;       // per-tile gather-index blocks in flight
constexpr int TREC_CONSUMERS = N_GATHER + 4 + 2;  // gather warps + epilogue warps + MMA + weight loader
constexpr int W_EPI0 = 8, W_MMA = 12, W_BLOAD = 13, W_SCHED = 14;

struct TileRec {
    int64_t row0;
    int rows, nt, list, dir, k, end, ncols, nsplit, ctr;
    uint32_t mask[4];
    uint8_t cols[128];        // active step columns (OS: dense offsets with a match; WS: {0})
    int32_t scatter[256];     // output row of each tile row (WS pairs; OS with os_rows)
};

struct ConvSmem {
    uint64_t full[16], empty[16], tfull[2], tempty[2];
    uint64_t trec_full[TREC_SLOTS], trec_empty[TREC_SLOTS];
    uint64_t blk_full[BLK_SLOTS], blk_empty[BLK_SLOTS];
    uint64_t claim_full[TREC_SLOTS], claim_empty[TREC_SLOTS];   // CTA pair: the leader's tile claims
    int64_t claim_v[TREC_SLOTS];                                 //   forwarded to the peer
    int started;                   // tiles the gather warps have begun (claim gate; shared atomics only)
    uint32_t tmem_holder[4];
    int tr, wsplit;                // device-chosen tile rows / weighted OS split active
    int n_sp;                      // tiles in the weighted split
    int64_t n_tiles;
    int sp_pre[SPLIT_MAX_TILES + 1];       // weighted split: first part of each tile (claim order)
    uint16_t sp_cnt[SPLIT_MAX_TILES];      // parts of each tile
    int epi_last[2];               // split-K fixup decisions, double-buffered by tile parity
    int list_prefix[SPC_MAX_KVOL + 1];
    TileRec trec[TREC_SLOTS];
};

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// OS split-K fixup, run by the 4 epilogue warps (thread = tile row within a 128-row half).
// Every part of an output tile red.adds its partial into the fp32 accumulator, releases
// its TMEM accumulator at once (the MMA warp moves on), then bumps the tile's arrival
// counter; the part that completes the count reads the sum back, adds the residual,
// writes the final dtype, and returns the accumulator rows and the counter to zero (so
// the next launch needs no zero-fill).
template <bool EPI>
__device__ __noinline__ void os_split_fixup(const ConvParams &p, ConvSmem &cs, const TileRec &R, uint32_t ti,
                                            int split, int nht, uint32_t tmem_tile, uint32_t tempty_bar, int e,
                                            int lane) {
    const int fl = ti & 1;
    const bool lead = threadIdx.x == 32 * W_EPI0;
    int *ctr = p.tile_ctr + R.ctr;
    if (R.ncols > 0) {
        const int ncc = (p.BN + 31) / 32;
        for (int h = 0; h < nht; ++h) {
            const int r = h * TC_BM + e * 32 + lane;
            const uint32_t tb = tmem_tile + h * p.tmem_cols + ((uint32_t)(e * 32) << 16);
            for (int cc = 0; cc < ncc; ++cc) {
                const int col = ((cc + R.list) % ncc) * 32;   // parts of a tile start on different columns
                uint32_t v[32];
                const int n = min(32, p.BN - col);
                if (n == 32) ptx::tmem_ld32(tb + col, v);
                else ptx::tmem_ld16(tb + col, v);
                ptx::tmem_ld_wait();
                if (r < R.rows) {
                    float *op = p.acc + (R.row0 + r) * p.ld_acc + R.nt * p.BN + col;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (q * 4 < n)
                            ptx::red_add_v4(op + 4 * q, to_f(v[4 * q]), to_f(v[4 * q + 1]), to_f(v[4 * q + 2]),
                                            to_f(v[4 * q + 3]));
                }
            }
        }
    }
    // TMEM no longer needed: hand the accumulator back to the MMA warp
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(tempty_bar);
    // release: the barrier orders the 128 threads' reductions before the lead's
    // gpu-scope fence (cumulative), then the arrival count
    epi_bar();
    if (lead) {
        __threadfence();
        const int old = atomicAdd(ctr, 1);
        __threadfence();
        cs.epi_last[fl] = old == split - 1;
    }
    epi_bar();
    if (!cs.epi_last[fl]) return;
    for (int h = 0; h < nht; ++h) {
        const int r = h * TC_BM + e * 32 + lane;
        if (r >= R.rows) continue;
        const int64_t row = R.row0 + r;   // accumulator row (tile order)
        const int64_t orow = p.os_rows ? (int64_t)R.scatter[r] : row;
        for (int col = 0; col < p.BN; col += 32) {
            uint32_t v[32];
            const int n = min(32, p.BN - col);
            const int gcol = R.nt * p.BN + col;
            float4 *ap = reinterpret_cast<float4 *>(p.acc + row * p.ld_acc + gcol);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q * 4 < n) {
                    const float4 s4 = __ldcg(ap + q);
                    v[4 * q] = __float_as_uint(s4.x);
                    v[4 * q + 1] = __float_as_uint(s4.y);
                    v[4 * q + 2] = __float_as_uint(s4.z);
                    v[4 * q + 3] = __float_as_uint(s4.w);
                    __stcg(ap + q, make_float4(0.f, 0.f, 0.f, 0.f));
                }
            if constexpr (EPI) {
                if (p.epi.scale || p.epi.shift) epi_affine_u32(p.epi, v, gcol, n);
            }
            store_row<EPI>(p, orow, gcol, v, n);
        }
    }
    if (lead) *reinterpret_cast<volatile int *>(ctr) = 0;
}

// one pipeline stage of the gather: nin slices (offset column, channel chunk) x NBT*RPI*8
// rows.  lane -> (row r_in of an RPI-row block, 16-byte chunk q_lane); every warp
// instruction stores whole sectors of RPI rows into the swizzled K-major tile (chunk j of
// row r lands at j ^ f(r)).  Matched rows: one whole-line request per row; sentinel rows
// (no input voxel) never touch L2: zeroed with a shared store.
// (ci, cc): offset column and channel chunk of the stage's first slice, advanced per slice
// (no integer division in the loop)
template <int BK, int NBT>
__device__ __forceinline__ void gather_slices(const ConvParams &p, const TileRec &R, uint32_t Bs, int kd, int rows,
                                              int ci, int cc, int nin, uint32_t abase, uint32_t kb_a, int warp,
                                              int r_in, int q_lane) {
    constexpr uint32_t rb = BK * 2;
    constexpr int RPI = 32 / (BK / 8);
    constexpr int ROWS_W = NBT * RPI;
    for (int kb = 0; kb < nin; ++kb) {
        // all of a slice's gather indices are loaded (explicit ld.shared, independent)
        // before its copies are issued
        int32_t g[NBT];
        {
            const int c = p.mode == 0 ? R.cols[ci] : 0;
#pragma unroll
            for (int b = 0; b < NBT; ++b) {
                const int r = warp * ROWS_W + b * RPI + r_in;
                g[b] = r < rows ? ptx::lds_s32(Bs + (uint32_t)(r * kd + c) * 4u) : -1;
            }
        }
        const uint32_t kbo = kb * kb_a;
#pragma unroll
        for (int b = 0; b < NBT; ++b) {
            const int r = warp * ROWS_W + b * RPI + r_in;
            const uint32_t f = rb == 128 ? (r & 7) : (rb == 64 ? ((r >> 1) & 3) : ((r >> 2) & 1));
            const uint32_t so = kbo + (uint32_t)r * rb + ((q_lane ^ f) * 16);
            // sentinel rows (no input voxel) never touch L2: a shared store of zeros
            // (measured faster than a src-size-0 cp.async zero fill on the level-0 layers)
            if (g[b] >= 0)
                ptx::cp_async_16(abase + so, p.f_in + (int64_t)g[b] * p.ld_in_bytes + cc * rb + q_lane * 16, 16u);
            else
                asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(abase + so), "r"(0) : "memory");
        }
        if (++cc == p.n_chunks) {
            cc = 0;
            ++ci;
        }
    }
}

// gather producer warps: per tile, wait for its record and index block, then fill the
// stages with (offset column, channel chunk) slices; a stage holds up to nkb consecutive
// slices (several chunks of one offset, or several offsets)
template <int BK, int NBT>
__device__ __forceinline__ void gather_role(const ConvParams &p, ConvSmem &cs, const int32_t *blk, int blk_stride, int kd,
                                            uint8_t *sa, int S, int nkb, uint32_t a_bytes, uint32_t kb_a, int warp,
                                            int lane) {
    constexpr int RPI = 32 / (BK / 8);         // rows per warp instruction (4 / 8 / 16)
    const int r_in = lane % RPI, q_lane = lane / RPI;
    int s = 0;
    uint32_t ph = 0;   // stage ring position / phase
    for (uint32_t ti = 0;; ++ti) {
        const int st = ti % TREC_SLOTS;
        ptx::mbar_wait(ptx::smem_u32(&cs.trec_full[st]), (ti / TREC_SLOTS) & 1);
        const TileRec &R = cs.trec[st];
        if (R.end) break;
        if (warp == 0 && lane == 0) ptx::red_max_shared(ptx::smem_u32(&cs.started), (int)ti + 1);   // ordered flag
        const int rows = R.rows, ncols = R.ncols;
        const int bs = ti % p.blk_slots;
        ptx::mbar_wait(ptx::smem_u32(&cs.blk_full[bs]), (ti / p.blk_slots) & 1);
        const int32_t *B = blk + bs * blk_stride;
        const int nsl = ncols * p.n_chunks;
        int ci = 0, cc = 0;   // (offset column, channel chunk) of slice sl
        for (int sl = 0; sl < nsl; sl += nkb) {
            const int nin = min(nkb, nsl - sl);
            ptx::mbar_wait(ptx::smem_u32(&cs.empty[s]), ph ^ 1);
            gather_slices<BK, NBT>(p, R, ptx::smem_u32(B), kd, rows, ci, cc, nin, ptx::smem_u32(sa + (size_t)s * a_bytes),
                                   kb_a, warp, r_in, q_lane);
            for (int k = 0; k < nin; ++k)
                if (++cc == p.n_chunks) {
                    cc = 0;
                    ++ci;
                }
            // the zero rows were written through the generic proxy: order them before the
            // tensor core's async-proxy reads, then arrive once this thread's copies land
            ptx::fence_proxy_async();
            ptx::cp_async_mbar_arrive(ptx::smem_u32(&cs.full[s]));
            if (++s == S) { s = 0; ph ^= 1; }
        }
        __syncwarp();
        if (lane == 0) {
            ptx::mbar_arrive(ptx::smem_u32(&cs.blk_empty[bs]));
            ptx::mbar_arrive(ptx::smem_u32(&cs.trec_empty[st]));
        }
    }
    ptx::cp_async_wait<0>();
}

// epilogue warps (8-11, thread = TMEM lane = tile row): TMEM -> OS: plain stores (final
// dtype, fused residual, or fp32 accumulator) / WS: red.global.add.v4.f32 scatter;
// FIX: OS split tiles go through the split-K fixup instead
constexpr int RED_COLS = 64;      // WS scatter: columns per bulk reduction (256-byte row segments)
constexpr int RED_LD = RED_COLS + 4;   // floats per staging row (16-byte aligned, fewer bank conflicts)
constexpr int RED_STAGE_BYTES = 4 * 32 * RED_LD * 4;

template <bool FIX, bool EPI>
__device__ __forceinline__ void epi_role(const ConvParams &p, ConvSmem &cs, float *red_stage, uint32_t tmem_base,
                                         int tr, int nht, int NH, int warp, int lane, int pair_rank) {
    const int e = warp - W_EPI0;   // == warp % 4: the TMEM lane quadrant this warp may access
    // WS scatter through bulk reductions (cp.reduce.async.bulk .add.f32, TMA engine): each
    // lane stages its row's 64-column segment in shared memory and reduces it into the fp32
    // accumulator in one operation -- measured 1.5-2x the red.global.add.v4 rate, which
    // is bound by one L2 transaction per lane and 16 bytes (scripts/red_bench.cu)
    const bool bulk = p.out_kind == OUT_F32_RED && red_stage != nullptr;
    const uint32_t stg_row = bulk ? ptx::smem_u32(red_stage + (e * 32 + lane) * RED_LD) : 0u;
    for (uint32_t ti = 0;; ++ti) {
        const int st = ti % TREC_SLOTS;
        ptx::mbar_wait_sleep(ptx::smem_u32(&cs.trec_full[st]), (ti / TREC_SLOTS) & 1);
        const TileRec &R = cs.trec[st];
        if (R.end) break;
        const uint32_t a = ti % p.tbufs;
        const int nt = R.nt;
        ptx::mbar_wait_sleep(ptx::smem_u32(&cs.tfull[a]), (ti / p.tbufs) & 1);
        ptx::tc_fence_after();
        const bool fix = FIX && R.nsplit > 1;
        if (fix) {
            os_split_fixup<EPI>(p, cs, R, ti, R.nsplit, nht, tmem_base + a * NH * p.tmem_cols, ptx::smem_u32(&cs.tempty[a]),
                           e, lane);
        } else {
#pragma unroll 1
            for (int h = 0; h < nht; ++h) {
                const int r = h * TC_BM + e * 32 + lane;
                int64_t orow = -1;
                if (r < R.rows && R.ncols > 0)
                    orow = (p.mode == 0 && !p.os_rows) ? R.row0 + r : (int64_t)R.scatter[r];
                const uint32_t tbase = tmem_base + (a * NH + h) * p.tmem_cols + ((uint32_t)(e * 32) << 16);
                if (bulk) {
                    for (int c0 = 0; c0 < p.BN; c0 += RED_COLS) {
                        ptx::bulk_wait_read0();   // the previous segment's reduction has read the row
#pragma unroll
                        for (int sub = 0; sub < RED_COLS; sub += 32) {
                            uint32_t vals[32];
                            ptx::tmem_ld32(tbase + c0 + sub, vals);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(stg_row + (sub + 4 * q) * 4),
                                             "r"(vals[4 * q]), "r"(vals[4 * q + 1]), "r"(vals[4 * q + 2]),
                                             "r"(vals[4 * q + 3])
                                             : "memory");
                        }
                        ptx::fence_proxy_async();   // the staged row is read by the async (bulk) proxy
                        if (orow >= 0) {
                            ptx::bulk_reduce_add_f32(static_cast<float *>(p.out) + orow * p.ld_out + nt * p.BN + c0,
                                                     stg_row, RED_COLS * 4);
                            ptx::bulk_commit();
                        }
                    }
                    continue;
                }
                for (int col = 0; col < p.BN; col += 32) {
                    uint32_t vals[32];
                    const int n = min(32, p.BN - col);
                    if (n == 32) ptx::tmem_ld32(tbase + col, vals);
                    else ptx::tmem_ld16(tbase + col, vals);
                    ptx::tmem_ld_wait();
                    if (orow >= 0) {
                        const int gcol = nt * p.BN + col;
                        if (p.out_kind == OUT_F32_RED) {
                            float *op = static_cast<float *>(p.out) + orow * p.ld_out + gcol;
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                if (q * 4 < n)
                                    ptx::red_add_v4(op + 4 * q, to_f(vals[4 * q]), to_f(vals[4 * q + 1]),
                                                    to_f(vals[4 * q + 2]), to_f(vals[4 * q + 3]));
                        } else {
                            if constexpr (EPI) {
                                if (p.out_kind == OUT_FINAL && (p.epi.scale || p.epi.shift))
                                    epi_affine_u32(p.epi, vals, gcol, n);
                            }
                            store_row<EPI>(p, orow, gcol, vals, n);
                        }
                    }
                }
            }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (threadIdx.x == 32 * W_EPI0) trace_tile_event(p.trace, 6, ti);
        if (lane == 0) {
            // the accumulator is free again: a CTA pair's MMAs are issued by the leader, so
            // the peer releases the leader's barrier
            if (pair_rank == 1) ptx::mbar_arrive_remote_relaxed(ptx::mapa(ptx::smem_u32(&cs.tempty[a]), 0));
            else if (!fix) ptx::mbar_arrive(ptx::smem_u32(&cs.tempty[a]));   // (the fixup released it already)
            ptx::mbar_arrive(ptx::smem_u32(&cs.trec_empty[st]));
        }
    }
    if (bulk) ptx::bulk_wait0();   // every reduction has landed before the CTA exits
}

// fp32 accumulator rows -> output dtype (+ residual), 8 columns per work item; the
// accumulator is returned to zero (workspace invariant).
__device__ __forceinline__ void convert_items(float *__restrict__ acc, int64_t ld_acc, int64_t n, int c_out, int out_dtype,
                                              void *__restrict__ out, int64_t ld_out, const void *__restrict__ res,
                                              int64_t ld_res, int clear, int64_t first, int64_t stride,
                                              const Epi &epi) {
    const bool ep = epi_on(epi);
    const int g8 = c_out / 8;                 // c_out is a multiple of 16
    const int64_t total = n * g8;
    for (int64_t e = first; e < total; e += stride) {
        const int64_t r = e / g8;
        const int c = (int)(e - r * g8) * 8;
        float4 *ap = reinterpret_cast<float4 *>(acc + r * ld_acc + c);
        const float4 a0 = __ldcg(ap), a1 = __ldcg(ap + 1);
        if (clear) {
            __stcg(ap, make_float4(0.f, 0.f, 0.f, 0.f));
            __stcg(ap + 1, make_float4(0.f, 0.f, 0.f, 0.f));
        }
        float v[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        if (ep) epi_affine(epi, v, c);
        if (out_dtype == SPC_F32) {
            if (res) {
                const float4 b0 = *reinterpret_cast<const float4 *>(static_cast<const float *>(res) + r * ld_res + c);
                const float4 b1 = *reinterpret_cast<const float4 *>(static_cast<const float *>(res) + r * ld_res + c + 4);
                v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
                v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
            }
            if (ep) epi_relu(epi, v);
            float *o = static_cast<float *>(out) + r * ld_out + c;
            *reinterpret_cast<float4 *>(o) = make_float4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<float4 *>(o + 4) = make_float4(v[4], v[5], v[6], v[7]);
        } else {
            if (res) {
                const uint4 u = *reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(res) + r * ld_res + c);
                const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 f = unpack2(w[q], out_dtype);
                    v[2 * q] += f.x;
                    v[2 * q + 1] += f.y;
                }
            }
            if (ep) epi_relu(epi, v);
            *reinterpret_cast<uint4 *>(static_cast<uint16_t *>(out) + r * ld_out + c) =
                make_uint4(pack2(v[0], v[1], out_dtype), pack2(v[2], v[3], out_dtype), pack2(v[4], v[5], out_dtype),
                           pack2(v[6], v[7], out_dtype));
        }
    }
}

template <int BK, int BM, int CG, bool EPI = false>
__global__ void __launch_bounds__(TC_THREADS, 1) k_conv_tc(const __grid_constant__ ConvParams p) {
    constexpr int NH = BM / TC_BM;   // 128-row MMA halves per tile (per CTA)
    static_assert(CG == 1 || BM == TC_BM, "a CTA of a pair holds 128 rows");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // stage buffers need 1024-byte alignment (swizzle atoms)
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // layout: [ring: S x A stage][S x B stage] ... [ConvSmem][gather-index blocks]; the ring
    // is carved per tile height below, the header sits after the largest carve
    ConvSmem &cs = *reinterpret_cast<ConvSmem *>(smem + p.hdr_off);
    // gather-index blocks: OS: the tile's [rows x k_dense] slice of the OS table (one bulk
    // copy per tile); WS: the 128 gather indices of the tile's pairs
    const int kd = p.mode == 0 ? p.k_dense : 1;
    int32_t *blk = reinterpret_cast<int32_t *>(smem + p.hdr_off + ((sizeof(ConvSmem) + 127) & ~size_t(127)));
    const int blk_stride = (BM * kd + 3) & ~3;      // int32 per block (16-byte multiple)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // CTA pair (cta_group::2): rank 0 issues the MMAs of both CTAs; rank 1 forwards its
    // stage completions and accumulator releases to rank 0's barriers
    const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0u;
    const bool leader = rank == 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < 16; ++s) {
            // gather threads + weight expect_tx (+ the peer's forwarded stage on a pair's leader)
            ptx::mbar_init(ptx::smem_u32(&cs.full[s]), N_GATHER * 32 + 1 + (CG == 2 && leader ? 1 : 0));
            ptx::mbar_init(ptx::smem_u32(&cs.empty[s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(ptx::smem_u32(&cs.tfull[a]), 1);
            ptx::mbar_init(ptx::smem_u32(&cs.tempty[a]), 4 + (CG == 2 && leader ? 4 : 0));
        }
        for (int i = 0; i < TREC_SLOTS; ++i) {
            ptx::mbar_init(ptx::smem_u32(&cs.trec_full[i]), 32);
            ptx::mbar_init(ptx::smem_u32(&cs.trec_empty[i]), TREC_CONSUMERS);
        }
        for (int i = 0; i < BLK_SLOTS; ++i) {
            ptx::mbar_init(ptx::smem_u32(&cs.blk_full[i]), 32);
            ptx::mbar_init(ptx::smem_u32(&cs.blk_empty[i]), N_GATHER);
        }
        for (int i = 0; i < TREC_SLOTS; ++i) {
            ptx::mbar_init(ptx::smem_u32(&cs.claim_full[i]), 1);
            ptx::mbar_init(ptx::smem_u32(&cs.claim_empty[i]), 1);
        }
        cs.started = 0;
        ptx::fence_mbar_init();
        ptx::fence_proxy_async();
        trace_event(p.trace, 0, 0);
    }
    if (warp == W_MMA) {
        if constexpr (CG == 2) ptx::tmem_alloc2(ptx::smem_u32(cs.tmem_holder), p.tbufs * NH * p.tmem_cols);
        else ptx::tmem_alloc(ptx::smem_u32(cs.tmem_holder), p.tbufs * NH * p.tmem_cols);
    }
    // a pair's barriers are initialised before either CTA signals the other's
    if constexpr (CG == 2) ptx::cluster_sync();
    // everything above overlaps the previous kernel's tail (PDL).  With maps_ready (the
    // caller asserts that the kernel map and weights were complete before the previous
    // kernel of the stream started -- every layer after the first of a pass), the
    // scheduler decodes its first tile and fetches its index block and the weight loader
    // streams weights while the previous layer drains; the roles that read features, write
    // outputs or touch the workspace wait for the previous kernel first
    const bool early = p.maps_ready && (warp == W_SCHED || warp == W_BLOAD || warp == W_MMA);
    if (!early) pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) trace_event(p.trace, 1, 0);
    const int64_t n_out = dev_count(p.n_out_cap, p.n_out_dev);
    if (warp == W_SCHED) {
        // tile geometry from the live (device-side) counts, no host sync: 256-row tiles
        // only when they still give >= 2 tiles per SM, else 128-row tiles; an OS part
        // with fewer 128-row tiles than SMs splits each tile's offsets over CTAs
        // (split-K, reduced in the epilogue fixup below)
        if (p.mode == 0) {
            int tr = CG == 2 ? 256 : BM;   // a pair's tile: 256 rows, 128 per CTA
            if (CG == 1 && BM == 256 && ((n_out + 255) / 256) * p.n_ntiles < 2 * p.num_sms) tr = 128;
            if (CG == 1 && p.force_tr) tr = min(p.force_tr, BM);
            const int64_t rt = (n_out + tr - 1) / tr;
            // weighted split-K for small launches (parts computed by the scheduler role)
            // (only when tiles leave at least half the SMs idle: the parts' fp32 reductions
            // land in one burst at the end of the launch and cost more than mild imbalance)
            const bool wsplit = CG == 1 && p.split_ok && p.k_dense >= 4 &&
                                2 * rt * p.n_ntiles <= p.split_tiles_per_sm2 && rt <= SPLIT_MAX_TILES &&
                                p.n_ntiles <= 2;
            const int64_t units = rt;
            if (lane == 0) {
                cs.tr = tr;
                cs.wsplit = wsplit ? 1 : 0;
                cs.n_sp = (int)rt;
                cs.n_tiles = units * p.n_ntiles;
            }
        } else {
            // virtual-tile prefix over the WS lists
            auto scan = [&](int tr, bool write) {
                int carry = 0;
                for (int base = 0; base < p.n_lists; base += 32) {
                    const int l = base + lane;
                    int v = 0;
                    if (l < p.n_lists && l != p.skip_list) {
                        const int cnt = p.counts[SPC_MAX_KVOL + l];
                        v = ((cnt + tr - 1) / tr) * (p.list_mirror[l] ? 2 : 1);
                    }
                    int x = v;
                    for (int o = 1; o < 32; o <<= 1) {
                        int y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                    }
                    if (write && l < p.n_lists) cs.list_prefix[l] = carry + x - v;
                    carry += __shfl_sync(0xffffffffu, x, 31);
                }
                return carry;
            };
            int tr = CG == 2 ? 256 : BM;
            if (CG == 1 && BM == 256 && (int64_t)scan(256, false) * p.n_ntiles < 2 * p.num_sms) tr = 128;
            if (CG == 1 && p.force_tr) tr = min(p.force_tr, BM);
            const int total = scan(tr, true);
            if (lane == 0) {
                cs.list_prefix[p.n_lists] = total;
                cs.tr = tr;
                cs.wsplit = 0;
                cs.n_tiles = (int64_t)total * p.n_ntiles;
            }
        }
        __syncwarp();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = cs.tmem_holder[0];
    if (threadIdx.x == 0) trace_event(p.trace, 2, 0);
    constexpr uint32_t rb = BK * 2;           // bytes per operand row (= swizzle span)
    // tr: rows of a tile (a pair's tile for CG = 2); nht: 128-row MMA halves held by this CTA
    const int tr = cs.tr, wsplit = cs.wsplit, nht = CG == 2 ? 1 : tr / TC_BM;
    // the ring carve of this tile height
    const int rgi = (BM == 256 && tr == 128) ? 1 : 0;
    const int S = p.ring[rgi].stages, nkb = p.ring[rgi].nkb;
    const uint32_t kb_a = p.ring[rgi].kb_a, a_bytes = p.ring[rgi].a_bytes, b_bytes = p.ring[rgi].b_bytes;
    uint8_t *sa = smem;
    uint8_t *sb = sa + (size_t)S * a_bytes;

    if (warp == W_SCHED) {
        // ===================== scheduler: tile records + gather indices ==================
        int64_t n_tiles = cs.n_tiles;
        if (wsplit) {
            // tile t (claim order, heaviest first) of w_t active offsets runs as
            // ceil(w_t / U) parts, U = ceil(total / SMs) (>= 2); weights precomputed by the
            // density-order pass, else popcounts of the tile masks
            const int64_t rt = cs.n_sp;
            const int f = tr / 128;
            const int64_t nt128 = (n_out + 127) / 128;
            const int32_t *wpre = p.tile_order ? p.tile_order + 2 * p.tiles128_cap + (tr == 256 ? p.tiles128_cap : 0) : nullptr;
            int wsum = 0;
#pragma unroll 4
            for (int t = lane; t < rt; t += 32) {
                int w = 0;
                if (wpre) {
                    w = wpre[t];
                } else {
                    for (int q = 0; q < p.tile_words; ++q) {
                        uint32_t m = 0;
                        for (int h = 0; h < f; ++h)
                            if (t * f + h < nt128) m |= p.tile_mask[(t * f + h) * p.tile_words + q];
                        w += __popc(m);
                    }
                }
                w = max(w, 1);
                cs.sp_cnt[t] = (uint16_t)w;
                wsum += w;
            }
            for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
            const int U = max(p.split_min_unit, (int)((wsum * (int64_t)p.n_ntiles + p.num_sms - 1) / p.num_sms));
            __syncwarp();
            int carry = 0;
            for (int base = 0; base < rt; base += 32) {
                const int t = base + lane;
                int c = 0;
                if (t < rt) {
                    const int w = cs.sp_cnt[t];
                    c = min((w + U - 1) / U, w);
                    cs.sp_cnt[t] = (uint16_t)c;
                }
                int x = c;
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (t < rt) cs.sp_pre[t] = carry + x - c;
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
            __syncwarp();
            n_tiles = (int64_t)carry * p.n_ntiles;
        }
        // tiles are claimed dynamically from a ws counter (heaviest first after the density
        // order), so uneven tiles balance across SMs; static round-robin without a ws
        int *fetch = p.tile_ctr ? p.tile_ctr + CTR_FETCH : nullptr;
        uint32_t ti = 0;
        // a pair's tiles: the leader claims (or walks statically without a ws) and forwards
        // every tile index to the peer, so both CTAs decode the same sequence
        const int64_t v_first = CG == 2 ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
        const int64_t v_step = CG == 2 ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;
        for (int64_t vs = v_first;; vs += v_step, ++ti) {
            const int st = ti % TREC_SLOTS;
            ptx::mbar_wait_sleep(ptx::smem_u32(&cs.trec_empty[st]), ((ti / TREC_SLOTS) & 1) ^ 1);
            int64_t v = vs;
            if (CG == 2 && !leader) {
                ptx::mbar_wait_cluster(ptx::smem_u32(&cs.claim_full[st]), (ti / TREC_SLOTS) & 1);
                v = *reinterpret_cast<volatile int64_t *>(&cs.claim_v[st]);
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_remote_relaxed(ptx::mapa(ptx::smem_u32(&cs.claim_empty[st]), 0));
            } else if (fetch && ti > 0) {
                if (ti == 1 && p.maps_ready) pdl_wait();   // the fetch counter is shared with the previous layer
                // first tile: blockIdx.x (no claim latency); then claims from the counter,
                // at most claim_ahead tiles beyond the one the gather warps are on (claim
                // gate: keeps the dynamic balance while the record of a light tile is ready
                // before the gather warps finish the previous one)
                {
                    const int need = (int)ti + 1 - p.claim_ahead;
                    uint32_t ns = 32;
                    while (ptx::atom_add_shared(ptx::smem_u32(&cs.started), 0) < need) {
                        __nanosleep(ns);
                        if (ns < 256) ns <<= 1;
                    }
                }
                int x = 0;
                if (lane == 0) x = atomicAdd(fetch, 1);
                v = v_step + __shfl_sync(0xffffffffu, x, 0);
            }
            if (CG == 2 && leader) {
                ptx::mbar_wait(ptx::smem_u32(&cs.claim_empty[st]), ((ti / TREC_SLOTS) & 1) ^ 1);
                if (lane == 0) {
                    ptx::st_cluster_s64(ptx::mapa(ptx::smem_u32(&cs.claim_v[st]), 1), v);
                    ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(&cs.claim_full[st]), 1));
                }
                __syncwarp();
            }
            TileRec &R = cs.trec[st];
            if (v >= n_tiles) {
                if (lane == 0) R.end = 1;
                ptx::mbar_arrive(ptx::smem_u32(&cs.trec_full[st]));
                break;
            }
            TileInfo t;
            decode_tile(p, v, cs.list_prefix, n_out, tr, wsplit ? cs.sp_pre : nullptr, cs.sp_cnt, cs.n_sp, t);
            if constexpr (CG == 2) {
                // the pair's active offsets span all 256 rows; this CTA takes rows
                // [128 rank, 128 rank + 128) of the tile (maybe none in a ragged tail)
                if (p.mode == 0) decode_tile_mask(p, t);
                t.row0 += 128 * rank;
                t.rows = max(0, min(128, t.rows - 128 * (int)rank));
            }
            // the tile's gather indices first (they depend only on its rows): the block's
            // load overlaps the record's mask / column / scatter work below
            const int bs = ti % p.blk_slots;
            ptx::mbar_wait_sleep(ptx::smem_u32(&cs.blk_empty[bs]), ((ti / p.blk_slots) & 1) ^ 1);
            int32_t *B = blk + bs * blk_stride;
            const uint32_t fb = ptx::smem_u32(&cs.blk_full[bs]);
            if (p.mode == 0) {
                // OS: rows [row0, row0+rows) of the [n_out x k_dense] table are contiguous
                const uint32_t bytes = (uint32_t)((t.rows * p.k_dense * 4 + 15) & ~15);
                if (lane == 0 && bytes) {
                    ptx::mbar_arrive_expect_tx(fb, bytes);
                    ptx::bulk_g2s(ptx::smem_u32(B), p.os + t.row0 * p.k_dense, bytes, fb);
                }
                if (lane != 0 || !bytes) ptx::mbar_arrive(fb);
            }
            // output-row scatter values (WS pairs / OS density order) are loaded before the
            // mask is consumed, so the two round trips overlap
            constexpr int SCN = BM / 32;
            int32_t sc[SCN], gx[SCN];
            if (p.mode == 1) {
                const int2 *pr = p.pairs + t.list * p.list_stride + t.row0;
#pragma unroll
                for (int q = 0; q < SCN; ++q) {
                    const int r = q * 32 + lane;
                    const int2 pq = r < t.rows ? pr[r] : make_int2(-1, -1);
                    sc[q] = t.dir ? pq.x : pq.y;
                    gx[q] = t.dir ? pq.y : pq.x;
                }
            } else if (p.os_rows) {
#pragma unroll
                for (int q = 0; q < SCN; ++q) {
                    const int r = q * 32 + lane;
                    sc[q] = (r < tr && r < t.rows) ? p.os_rows[t.row0 + r] : -1;
                }
            }
            if (CG == 1 && p.mode == 0) decode_tile_mask(p, t);
            // active columns: warp-parallel compaction of the mask bits (ballot prefix),
            // then this part's contiguous share when the tile is split
            int nc = 0;
            {
                int c0 = 0, c1 = 128;
                int total = 0;
#pragma unroll
                for (int w = 0; w < 4; ++w) total += __popc(t.mask[w]);
                if (p.mode == 0 && t.nsplit > 1) {
                    const int per = (total + t.nsplit - 1) / t.nsplit;
                    c0 = min(total, t.list * per);
                    c1 = min(total, c0 + per);
                }
                int base = 0;
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const uint32_t bits = t.mask[w];
                    const int pos = base + __popc(bits & ptx_lanemask_lt());
                    if (((bits >> lane) & 1u) && pos >= c0 && pos < c1) R.cols[pos - c0] = (uint8_t)(w * 32 + lane);
                    base += __popc(bits);
                }
                nc = max(0, min(total, c1) - c0);
            }
            if (lane == 0) {
                R.row0 = t.row0; R.rows = t.rows; R.nt = t.nt; R.list = t.list; R.dir = t.dir; R.k = t.k; R.end = 0;
                R.nsplit = p.mode == 0 ? t.nsplit : 1;
                R.ctr = t.ctr;
                for (int w = 0; w < 4; ++w) R.mask[w] = t.mask[w];
                R.ncols = nc;
            }
            if (p.mode == 1) {
#pragma unroll
                for (int q = 0; q < SCN; ++q) {
                    R.scatter[q * 32 + lane] = sc[q];
                    B[q * 32 + lane] = gx[q];
                }
                ptx::mbar_arrive(fb);
            } else if (p.os_rows) {
#pragma unroll
                for (int q = 0; q < SCN; ++q)
                    if (q * 32 < tr) R.scatter[q * 32 + lane] = sc[q];
            }
            ptx::mbar_arrive(ptx::smem_u32(&cs.trec_full[st]));
            if (lane == 0) trace_tile_event(p.trace, 3, ti);
        }
        ptx::cp_async_wait<0>();
    } else if (warp < N_GATHER) {
        // ===================== gather producers (cp.async, 8 warps) =====================
        // one loop per tile height (row blocks per warp fixed at compile time)
        constexpr int NB = BM / N_GATHER / (32 / (BK / 8));
        if (NB > 1 && tr < BM)
            gather_role<BK, (NB > 1 ? NB / 2 : 1)>(p, cs, blk, blk_stride, kd, sa, S, nkb, a_bytes, kb_a, warp, lane);
        else
            gather_role<BK, NB>(p, cs, blk, blk_stride, kd, sa, S, nkb, a_bytes, kb_a, warp, lane);
    } else if (warp == W_BLOAD) {
        // ===================== weight loader (1-D bulk copies, TMA engine) ===============
        int s = 0;
        uint32_t ph = 0;   // stage ring position / phase (no division per stage)
        for (uint32_t ti = 0;; ++ti) {
            const int st = ti % TREC_SLOTS;
            ptx::mbar_wait(ptx::smem_u32(&cs.trec_full[st]), (ti / TREC_SLOTS) & 1);
            const TileRec &R = cs.trec[st];
            if (R.end) break;
            if (lane == 0) {
                const int nt = R.nt, kfix = R.k, ncols = R.ncols;
                const int nsl = ncols * p.n_chunks;
                int ci = 0, cc = 0;   // (offset column, channel chunk) of the next slice
                for (int sl = 0; sl < nsl; sl += nkb) {
                    const int nin = min(nkb, nsl - sl);
                    ptx::mbar_wait(ptx::smem_u32(&cs.empty[s]), ph ^ 1);
                    const uint32_t fb = ptx::smem_u32(&cs.full[s]);
                    // a CTA of a pair loads its N half of each weight tile (rows
                    // [rank BN/2, (rank+1) BN/2) of the K-major blob: contiguous, atom-aligned)
                    const uint32_t kb_bl = p.kb_b / CG;
                    ptx::mbar_arrive_expect_tx(fb, nin * kb_bl);
                    for (int kb = 0; kb < nin; ++kb) {
                        const int k = p.mode == 0 ? p.dense_k[R.cols[ci]] : kfix;
                        const int64_t blob = ((int64_t)k * p.n_ntiles + nt) * p.n_chunks + cc;
                        ptx::bulk_g2s(ptx::smem_u32(sb + (size_t)s * b_bytes + kb * kb_bl),
                                      p.wblob + blob * p.kb_b + rank * kb_bl, kb_bl, fb);
                        if (++cc == p.n_chunks) {
                            cc = 0;
                            ++ci;
                        }
                    }
                    if (++s == S) { s = 0; ph ^= 1; }
                }
                ptx::mbar_arrive(ptx::smem_u32(&cs.trec_empty[st]));
            }
            __syncwarp();
        }
    } else if (CG == 2 && warp == W_MMA && !leader) {
        // ===================== pair peer: stage forwarder =====================================
        // the leader's MMAs read this CTA's A rows and B half: once a stage is complete here,
        // make it visible to the async proxy and arrive on the leader's full barrier
        int s = 0;
        uint32_t ph = 0;
        for (uint32_t ti = 0;; ++ti) {
            const int st = ti % TREC_SLOTS;
            ptx::mbar_wait(ptx::smem_u32(&cs.trec_full[st]), (ti / TREC_SLOTS) & 1);
            const TileRec &R = cs.trec[st];
            if (__shfl_sync(0xffffffffu, R.end, 0)) break;
            const int nsl = __shfl_sync(0xffffffffu, R.ncols, 0) * p.n_chunks;
            for (int sl = 0; sl < nsl; sl += nkb) {
                ptx::mbar_wait(ptx::smem_u32(&cs.full[s]), ph);
                ptx::fence_proxy_async();
                if (lane == 0) ptx::mbar_arrive_remote_relaxed(ptx::mapa(ptx::smem_u32(&cs.full[s]), 0));
                if (++s == S) { s = 0; ph ^= 1; }
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&cs.trec_empty[st]));
        }
    } else if (warp == W_MMA) {
        // ===================== MMA issuer (whole warp, elected lane issues) ================
        // every lane runs the loop on warp-uniform values (shuffled from lane 0), so the
        // descriptors stay uniform and each tcgen05.mma is one predicated instruction
        int ring_s = 0;
        uint32_t ring_ph = 0;   // stage ring position / phase (no division per stage)
        const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base, 0);
        const uint32_t kb_a_u = __shfl_sync(0xffffffffu, kb_a, 0), a_bytes_u = __shfl_sync(0xffffffffu, a_bytes, 0);
        const uint32_t b_bytes_u = __shfl_sync(0xffffffffu, b_bytes, 0);
        const int S_u = __shfl_sync(0xffffffffu, S, 0), nkb_u = __shfl_sync(0xffffffffu, nkb, 0);
        const int nht_u = __shfl_sync(0xffffffffu, nht, 0);
        const uint32_t idesc_u = p.idesc;
        const uint32_t sa_u = __shfl_sync(0xffffffffu, ptx::smem_u32(sa), 0);
        const uint32_t sb_u = __shfl_sync(0xffffffffu, ptx::smem_u32(sb), 0);
        for (uint32_t ti = 0;; ++ti) {
            const int st = ti % TREC_SLOTS;
            ptx::mbar_wait(ptx::smem_u32(&cs.trec_full[st]), (ti / TREC_SLOTS) & 1);
            const TileRec &R = cs.trec[st];
            if (__shfl_sync(0xffffffffu, R.end, 0)) break;
            const int ncols = __shfl_sync(0xffffffffu, R.ncols, 0);
            const uint32_t a = ti % p.tbufs;
            ptx::mbar_wait(ptx::smem_u32(&cs.tempty[a]), ((ti / p.tbufs) & 1) ^ 1);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tb + a * NH * p.tmem_cols;
            uint32_t acc = 0;
            const int nsl = ncols * p.n_chunks;
            const uint32_t kb_bl = p.kb_b / CG;
            for (int sl = 0; sl < nsl; sl += nkb_u) {
                const int nin = min(nkb_u, nsl - sl);
                const int s = ring_s;
                ptx::mbar_wait(ptx::smem_u32(&cs.full[s]), ring_ph);
                if (++ring_s == S_u) { ring_s = 0; ring_ph ^= 1; }
                if (sl == 0 && lane == 0) trace_tile_event(p.trace, 4, ti);
                ptx::fence_proxy_async();
                ptx::tc_fence_after();
                // descriptors built once per stage; the K / row-half / slice steps add to
                // the 14-bit start-address field (shared addresses < 256 KB: no carry out)
                const uint64_t a_d0 = ptx::umma_desc_kmajor_sw(sa_u + (uint32_t)s * a_bytes_u, rb);
                const uint64_t b_d0 = ptx::umma_desc_kmajor_sw(sb_u + (uint32_t)s * b_bytes_u, rb);
                for (int kb = 0; kb < nin; ++kb) {
                    const uint64_t a_dk = a_d0 + ((kb * kb_a_u) >> 4), b_dk = b_d0 + ((kb * kb_bl) >> 4);
                    if constexpr (CG == 2) {
                        // one M = 256 MMA chain for the pair (A rows and B halves at the same
                        // smem offsets in both CTAs, accumulators at the same TMEM address)
                        ptx::mma2_f16_ss_chain<BK / 16>(d_tmem, a_dk, b_dk, idesc_u, acc);
                    } else {
                        // one asm block per 128-row half: the slice's BK/16 K steps
#pragma unroll
                        for (int h = 0; h < NH; ++h) {
                            if (h >= nht_u) break;
                            ptx::mma_f16_ss_chain<BK / 16>(d_tmem + h * p.tmem_cols, a_dk + ((h * TC_BM * rb) >> 4),
                                                           b_dk, idesc_u, acc);
                        }
                    }
                    acc = 1;
                }
                if constexpr (CG == 2) ptx::mma2_commit_multicast_elect(ptx::smem_u32(&cs.empty[s]));
                else ptx::mma_commit_elect(ptx::smem_u32(&cs.empty[s]));
            }
            if constexpr (CG == 2) ptx::mma2_commit_multicast_elect(ptx::smem_u32(&cs.tfull[a]));
            else ptx::mma_commit_elect(ptx::smem_u32(&cs.tfull[a]));
            if (lane == 0) trace_tile_event(p.trace, 5, ti);
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&cs.trec_empty[st]));
        }
    } else if (warp >= W_EPI0 && warp < W_EPI0 + 4) {
        // ===================== epilogue (warps 8-11, thread = TMEM lane = tile row) ====
        const int pair_rank = CG == 2 ? (int)rank : -1;
        float *red_stage = p.red_off ? reinterpret_cast<float *>(smem + p.red_off) : nullptr;
        if (wsplit)
            epi_role<true, EPI>(p, cs, red_stage, tmem_base, tr, nht, NH, warp, lane, pair_rank);
        else
            epi_role<false, EPI>(p, cs, red_stage, tmem_base, tr, nht, NH, warp, lane, pair_rank);
    }
    ptx::tc_fence_before();
    // a pair frees its TMEM and exits together (the leader's MMAs and commits reach the
    // peer's TMEM and barriers until its last tile)
    if constexpr (CG == 2) ptx::cluster_sync();
    else __syncthreads();
    if (warp == W_MMA) {
        ptx::tc_fence_after();
        if constexpr (CG == 2) ptx::tmem_dealloc2(tmem_base, p.tbufs * NH * p.tmem_cols);
        else ptx::tmem_dealloc(tmem_base, p.tbufs * NH * p.tmem_cols);
    }
    if (threadIdx.x == 0) trace_event(p.trace, 7, 0);
    if (p.tile_ctr && threadIdx.x == 0) {
        // the last CTA out returns the fetch / exit counters to zero (ws contract); every
        // CTA's scheduler has made its final claim before its CTA gets here
        __threadfence();
        if (atomicAdd(p.tile_ctr + CTR_EXIT, 1) == (int)gridDim.x - 1) {
            atomicExch(p.tile_ctr + CTR_FETCH, 0);
            atomicExch(p.tile_ctr + CTR_EXIT, 0);
        }
    }
}

// ------------------------------------------------------------------------------------
// fp32 FFMA path (same OS / WS semantics)
// ------------------------------------------------------------------------------------
constexpr int SM_TM = 64, SM_TN = 64, SM_TK = 16;

__global__ void __launch_bounds__(256) k_conv_simt(const __grid_constant__ ConvParams p, const float *__restrict__ W,
                                                   int c_in, int c_out) {
    __shared__ float As[SM_TK][SM_TM + 4];
    __shared__ float Bs[SM_TK][SM_TN];
    __shared__ int32_t gidx[SM_TM];
    __shared__ int64_t sidx[SM_TM];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    pdl_wait();
    pdl_trigger();
    const int64_t n_out = dev_count(p.n_out_cap, p.n_out_dev);
    const int col0 = blockIdx.y * SM_TN;
    int64_t row0;
    int rows, list = 0, dir = 0;
    int kfix = -1;
    if (p.mode == 0) {
        row0 = (int64_t)blockIdx.x * SM_TM;
        if (row0 >= n_out) return;
        rows = (int)imin64(SM_TM, n_out - row0);
    } else {
        // blockIdx.x -> (list, dir, tile) with a fixed per-list tile budget
        const int64_t tiles_per = (p.n_out_cap + SM_TM - 1) / SM_TM;
        const int64_t v = blockIdx.x;
        list = (int)(v / (2 * tiles_per));
        const int64_t rem = v - (int64_t)list * 2 * tiles_per;
        dir = (int)(rem / tiles_per);
        const int64_t tl = rem - (int64_t)dir * tiles_per;
        if (list >= p.n_lists) return;
        if (dir == 1 && !p.list_mirror[list]) return;
        const int cnt = p.counts[SPC_MAX_KVOL + list];
        row0 = tl * SM_TM;
        if (row0 >= cnt) return;
        rows = (int)imin64(SM_TM, cnt - row0);
        kfix = dir ? p.k_vol - 1 - p.list_k[list] : p.list_k[list];
    }
    float acc[4][4] = {};
    const int n_steps = p.mode == 0 ? p.k_dense : 1;
    for (int st = 0; st < n_steps; ++st) {
        const int k = p.mode == 0 ? p.dense_k[st] : kfix;
        __syncthreads();
        if (threadIdx.x < SM_TM) {
            const int r = threadIdx.x;
            int32_t g = -1;
            int64_t so = -1;
            if (r < rows) {
                if (p.mode == 0) {
                    g = p.os[(row0 + r) * p.k_dense + st];
                    so = p.os_rows ? p.os_rows[row0 + r] : row0 + r;
                } else {
                    const int2 pr = p.pairs[list * p.list_stride + row0 + r];
                    g = dir ? pr.y : pr.x;
                    so = dir ? pr.x : pr.y;
                }
            }
            gidx[r] = g;
            sidx[r] = so;
        }
        __syncthreads();
        for (int k0 = 0; k0 < c_in; k0 += SM_TK) {
            for (int e = threadIdx.x; e < SM_TM * SM_TK; e += 256) {
                const int r = e / SM_TK, kk = e % SM_TK;
                const int32_t g = gidx[r];
                As[kk][r] = (g >= 0 && k0 + kk < c_in)
                                ? reinterpret_cast<const float *>(p.f_in + (int64_t)g * p.ld_in_bytes)[k0 + kk]
                                : 0.f;
            }
            for (int e = threadIdx.x; e < SM_TK * SM_TN; e += 256) {
                const int kk = e / SM_TN, cc = e % SM_TN;
                Bs[kk][cc] = (k0 + kk < c_in && col0 + cc < c_out)
                                 ? W[((int64_t)k * c_in + k0 + kk) * c_out + col0 + cc]
                                 : 0.f;
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < SM_TK; ++kk) {
                float a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
            __syncthreads();
        }
    }
    for (int i = 0; i < 4; ++i) {
        const int r = ty * 4 + i;
        if (r >= rows) continue;
        const int64_t orow = sidx[r];
        for (int j = 0; j < 4; ++j) {
            const int col = col0 + tx * 4 + j;
            if (col >= c_out) continue;
            float v = acc[i][j];
            if (p.out_kind == OUT_FINAL) {
                if (p.epi.scale) v *= p.epi.scale[col];
                if (p.epi.shift) v += p.epi.shift[col];
            }
            if (p.out_kind == OUT_F32_RED) {
                atomicAdd(static_cast<float *>(p.out) + orow * p.ld_out + col, v);
            } else if (p.out_kind == OUT_F32_STORE || p.out_dtype == SPC_F32) {
                if (p.out_kind == OUT_FINAL && p.residual) v += static_cast<const float *>(p.residual)[orow * p.ld_res + col];
                if (p.out_kind == OUT_FINAL && p.epi.relu) v = fmaxf(v, 0.f);
                static_cast<float *>(p.out)[orow * p.ld_out + col] = v;
            } else {
                if (p.residual) {
                    const uint16_t h = static_cast<const uint16_t *>(p.residual)[orow * p.ld_res + col];
                    v += p.out_dtype == SPC_BF16 ? __bfloat162float(__ushort_as_bfloat16(h))
                                                 : __half2float(__ushort_as_half(h));
                }
                if (p.epi.relu) v = fmaxf(v, 0.f);
                static_cast<uint16_t *>(p.out)[orow * p.ld_out + col] =
                    p.out_dtype == SPC_BF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(v))
                                            : __half_as_ushort(__float2half_rn(v));
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// weight preparation, accumulator conversion, zero fill
// ------------------------------------------------------------------------------------
// weights -> per (k, N-tile, C-chunk) blobs laid out exactly as the swizzled K-major smem
// tile the MMA reads: row n (BK elements = rb bytes), 16-byte chunk j stored at j ^ f(n)
// mode (spc_weight_mode): 0 = W_k as given; 1 = W_k^T (c_in / c_out are those of the
// PREPARED weight: the source is [k_vol][c_out][c_in]); 2 = W_{k_vol-1-k}^T
__global__ void k_prepare_weight_tc(const uint16_t *__restrict__ w, int k_vol, int c_in, int c_out, int BK, int BN,
                                    int mode, uint16_t *__restrict__ out) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    const int64_t total = (int64_t)k_vol * c_in * c_out;
    const int n_nt = c_out / BN, n_ch = c_in / BK;
    const int rb = BK * 2;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int co = (int)(e % c_out);
        const int64_t t = e / c_out;
        const int ci = (int)(t % c_in);
        const int k = (int)(t / c_in);
        const int64_t src = mode == 0 ? e
                                      : ((int64_t)(mode == 2 ? k_vol - 1 - k : k) * c_out + co) * c_in + ci;
        const int nt = co / BN, n = co % BN, cc = ci / BK, c = ci % BK;
        const int64_t blob = ((int64_t)k * n_nt + nt) * n_ch + cc;
        const int f = rb == 128 ? (n & 7) : (rb == 64 ? ((n >> 1) & 3) : ((n >> 2) & 1));
        const int j = (c * 2) / 16, within = (c * 2) % 16;
        const int64_t byte = (int64_t)n * rb + (int64_t)((j ^ f) * 16) + within;
        out[blob * BN * BK + byte / 2] = w[src];
    }
}

// fp32 accumulator -> output dtype (+ residual): 8 columns per thread, 16/32-byte accesses
// clear != 0: the accumulator rows are returned to zero after the read (workspace invariant)
__global__ void k_convert(float *__restrict__ acc, int64_t ld_acc, int64_t n_cap, const int64_t *n_dev, int c_out,
                          int out_dtype, void *__restrict__ out, int64_t ld_out, const void *__restrict__ res,
                          int64_t ld_res, int clear, Epi epi) {
    pdl_wait();
    pdl_trigger();
    const int64_t n = dev_count(n_cap, n_dev);
    convert_items(acc, ld_acc, n, c_out, out_dtype, out, ld_out, res, ld_res, clear,
                  blockIdx.x * (int64_t)blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x, epi);
}

__global__ void k_zero_rows(float *__restrict__ acc, int64_t ld, int64_t n_cap, const int64_t *n_dev, int c) {
    pdl_wait();
    pdl_trigger();
    const int64_t n = dev_count(n_cap, n_dev);
    const int64_t total = n * c;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / c;
        acc[r * ld + (e - r * c)] = 0.f;
    }
}

static int pick_bk(int c_in) { return c_in % 64 == 0 ? 64 : (c_in % 32 == 0 ? 32 : 16); }
static int pick_bn(int c_out) {
    if (c_out <= 256) return c_out;
    for (int bn = 256; bn >= 16; bn -= 16)
        if (c_out % bn == 0) return bn;
    return 16;
}
static uint32_t pow2_cols(int n) {
    uint32_t c = 32;
    while ((int)c < n) c <<= 1;
    return c;
}

static size_t elem_size(int dt) { return dt == SPC_F32 ? 4 : 2; }

spc_status dense_forward(const void *f_in, int64_t ld_in, int in_dtype, int c_in, const void *wblob, int k, int c_out,
                         int BK, int BN, int64_t n_cap, const int64_t *n_dev, void *out, int64_t ld_out, int out_kind,
                         int out_dtype, const void *residual, int64_t ld_res, const Epi &epi,
                         cudaStream_t st);   // spc_dense.cu

}  // namespace spc

using namespace spc;

extern "C" size_t spc_prepared_weight_bytes(int32_t k_vol, int32_t c_in, int32_t c_out, int32_t in_dtype) {
    if (k_vol <= 0 || c_in <= 0 || c_out <= 0) return 0;
    return (size_t)k_vol * c_in * c_out * elem_size(in_dtype);
}

__global__ void k_transpose_weight_f32(const float *__restrict__ w, int k_vol, int c_in, int c_out, int mode,
                                       float *__restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const int64_t total = (int64_t)k_vol * c_in * c_out;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int co = (int)(e % c_out);
        const int64_t t = e / c_out;
        const int ci = (int)(t % c_in);
        const int k = (int)(t / c_in);
        out[e] = w[((int64_t)(mode == 2 ? k_vol - 1 - k : k) * c_out + co) * c_in + ci];
    }
}

// dst[r][0..c) += src[r][0..c) for the live rows (the residual branch of a backward pass);
// 8 columns per work item, c a multiple of 8, rows 16-byte aligned
__global__ void k_add_rows(void *__restrict__ dst, int64_t ld_dst, const void *__restrict__ src, int64_t ld_src,
                           int64_t n_cap, const int64_t *n_dev, int c, int dtype, int accumulate) {
    pdl_wait();
    pdl_trigger();
    const int64_t n = dev_count(n_cap, n_dev);
    const int g8 = c / 8;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * g8; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / g8;
        const int col = (int)(e - r * g8) * 8;
        if (dtype == SPC_F32) {
            float4 *d = reinterpret_cast<float4 *>(static_cast<float *>(dst) + r * ld_dst + col);
            const float4 *s = reinterpret_cast<const float4 *>(static_cast<const float *>(src) + r * ld_src + col);
            for (int q = 0; q < 2; ++q) {
                const float4 b = s[q];
                if (accumulate) {
                    float4 a = d[q];
                    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
                    d[q] = a;
                } else {
                    d[q] = b;
                }
            }
        } else {
            uint4 *d = reinterpret_cast<uint4 *>(static_cast<uint16_t *>(dst) + r * ld_dst + col);
            const uint4 u = *reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(src) + r * ld_src + col);
            if (!accumulate) {
                *d = u;
                continue;
            }
            const uint4 w = *d;
            const uint32_t a[4] = {w.x, w.y, w.z, w.w}, b[4] = {u.x, u.y, u.z, u.w};
            uint32_t o[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 x = unpack2(a[q], dtype), y = unpack2(b[q], dtype);
                o[q] = pack2(x.x + y.x, x.y + y.y, dtype);
            }
            *d = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
}

extern "C" spc_status spc_add_rows(void *dst, int64_t ld_dst, const void *src, int64_t ld_src, int64_t n_cap,
                                   const int64_t *n_dev, int32_t c, int32_t dtype, int32_t accumulate, void *stream) {
    SPC_CHECK_ARG(dst && src && c > 0 && c % 8 == 0 && ld_dst >= c && ld_src >= c, "bad arguments");
    SPC_CHECK_ARG(dtype >= SPC_F32 && dtype <= SPC_BF16, "bad dtype");
    const size_t es = dtype == SPC_F32 ? 4 : 2;
    SPC_CHECK_ARG((uintptr_t)dst % 16 == 0 && (uintptr_t)src % 16 == 0 && (ld_dst * es) % 16 == 0 &&
                      (ld_src * es) % 16 == 0,
                  "rows must be 16-byte aligned");
    if (n_cap == 0) return SPC_OK;
    const int64_t work = n_cap * (c / 8);
    SPC_CUDA(launch_pdl(k_add_rows, dim3((unsigned)std::min<int64_t>((work + 255) / 256, 8 * 148)), dim3(256), 0,
                        as_stream(stream), dst, ld_dst, src, ld_src, n_cap, n_dev, (int)c, (int)dtype,
                        accumulate ? 1 : 0));
    SPC_LAUNCH_CHECK("k_add_rows");
    return SPC_OK;
}

__global__ void k_bn_fold(const float *gamma, const float *beta, const float *mean, const float *var, float eps, int c,
                          float *scale, float *shift) {
    pdl_wait();
    pdl_trigger();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
        const float s = gamma[i] / sqrtf(var[i] + eps);
        scale[i] = s;
        shift[i] = beta[i] - mean[i] * s;
    }
}

extern "C" spc_status spc_bn_fold(const float *gamma, const float *beta, const float *mean, const float *var,
                                  float eps, int32_t c, float *scale, float *shift, void *stream) {
    SPC_CHECK_ARG(gamma && beta && mean && var && scale && shift && c > 0, "bad arguments");
    SPC_CUDA(launch_pdl(k_bn_fold, dim3((unsigned)((c + 255) / 256)), dim3(256), 0, as_stream(stream), gamma, beta,
                        mean, var, eps, (int)c, scale, shift));
    SPC_LAUNCH_CHECK("k_bn_fold");
    return SPC_OK;
}

extern "C" spc_status spc_prepare_weight(const void *weight, int32_t k_vol, int32_t c_in, int32_t c_out,
                                         int32_t in_dtype, void *prepared, void *stream) {
    return spc_prepare_weight_ex(weight, k_vol, c_in, c_out, in_dtype, SPC_WEIGHT_FORWARD, prepared, stream);
}

extern "C" spc_status spc_prepare_weight_ex(const void *weight, int32_t k_vol, int32_t c_in, int32_t c_out,
                                            int32_t in_dtype, int32_t mode, void *prepared, void *stream) {
    SPC_CHECK_ARG(weight && prepared, "null pointer");
    SPC_CHECK_ARG(k_vol >= 1 && k_vol <= SPC_MAX_KVOL && c_in > 0 && c_out > 0, "bad shape");
    SPC_CHECK_ARG(mode >= SPC_WEIGHT_FORWARD && mode <= SPC_WEIGHT_DGRAD_MIRROR, "bad weight mode");
    SPC_CHECK_ARG(weight != prepared, "weight and prepared must not alias");
    cudaStream_t st = as_stream(stream);
    // the kernels take the PREPARED layer's channel counts: a dgrad weight is that of a
    // (c_out -> c_in) layer
    if (mode != SPC_WEIGHT_FORWARD) std::swap(c_in, c_out);
    if (in_dtype == SPC_F32) {
        if (mode == SPC_WEIGHT_FORWARD) {
            SPC_CUDA(cudaMemcpyAsync(prepared, weight, (size_t)k_vol * c_in * c_out * 4, cudaMemcpyDeviceToDevice, st));
        } else {
            const int64_t total = (int64_t)k_vol * c_in * c_out;
            SPC_CUDA(launch_pdl(k_transpose_weight_f32, dim3((unsigned)std::min<int64_t>((total + 255) / 256, 4096)),
                                dim3(256), 0, st, static_cast<const float *>(weight), (int)k_vol, (int)c_in, (int)c_out,
                                (int)mode, static_cast<float *>(prepared)));
            SPC_LAUNCH_CHECK("k_transpose_weight_f32");
        }
        return SPC_OK;
    }
    SPC_CHECK_ARG(in_dtype == SPC_F16 || in_dtype == SPC_BF16, "bad dtype");
    if (c_in % 16 || c_out % 16)
        return fail(SPC_ERR_UNSUPPORTED, "spc_prepare_weight: f16/bf16 needs c_in and c_out multiples of 16");
    const int64_t total = (int64_t)k_vol * c_in * c_out;
    SPC_CUDA(launch_pdl(k_prepare_weight_tc, dim3((unsigned)std::min<int64_t>((total + 255) / 256, 4096)), dim3(256), 0, st, 
        static_cast<const uint16_t *>(weight), k_vol, c_in, c_out, pick_bk(c_in), pick_bn(c_out), (int)mode,
        static_cast<uint16_t *>(prepared)));
    SPC_LAUNCH_CHECK("k_prepare_weight_tc");
    return SPC_OK;
}

// ws layout: [fp32 accumulator n_out x c_out][256 int32 tile arrival counters]; both
// all-zero on entry and left all-zero on return (spc.h)
static constexpr size_t WS_CTR_BYTES = WS_CTR_SLOTS * sizeof(int);
extern "C" size_t spc_conv_workspace_size(const spc_kmap *km, int32_t c_out, int32_t out_dtype) {
    if (!km || c_out <= 0) return 0;
    (void)out_dtype;
    return align_up((size_t)km->n_out * c_out * 4, 256) + WS_CTR_BYTES;
}

static void fill_map_params(ConvParams &p, const spc_kmap *km) {
    // density-ordered OS part when the map has one (SPC_KMAP_DENSITY_ORDER)
    const bool ord = km->os_rows && km->os_table_ord && km->tile_mask_ord && option(SPC_OPT_CONV_DENSITY_ORDER) != 0;
    p.os = ord ? km->os_table_ord : km->os_table;
    p.os_rows = ord ? km->os_rows : nullptr;
    p.k_dense = km->k_dense;
    p.tile_mask = ord ? km->tile_mask_ord : km->tile_mask_dev;
    p.tile_order = ord ? km->tile_order : nullptr;
    p.tiles128_cap = (km->n_out + 127) / 128;
    p.tile_words = km->tile_words;
    p.pairs = reinterpret_cast<const int2 *>(km->ws_pairs);
    p.list_stride = km->n_out;
    p.counts = km->counts_dev;
    p.n_lists = km->n_lists;
    p.k_vol = km->k_vol;
    p.n_out_cap = km->n_out;
    p.n_out_dev = km->n_out_dev;
    for (int c = 0; c < km->k_dense; ++c) p.dense_k[c] = km->dense_k[c];
    for (int l = 0; l < km->n_lists; ++l) {
        p.list_k[l] = km->list_k[l];
        p.list_mirror[l] = km->list_mirror[l];
    }
}

static spc_status launch_tc(const ConvParams &p0, int mode, int out_kind, void *out, int64_t ld_out, cudaStream_t st) {
    ConvParams p = p0;
    p.mode = mode;
    p.out_kind = out_kind;
    p.out = out;
    p.ld_out = ld_out;
    const int kd = mode == 0 ? p.k_dense : 1;
    const size_t blk_bytes = (size_t)((p.bm * kd + 3) & ~3) * 4;
    const bool bulk_red = out_kind == OUT_F32_RED && p.BN % RED_COLS == 0 && option(SPC_OPT_CONV_BULK_RED) != 0;
    // slices (one BK-channel chunk of one offset) per pipeline stage: a stage carries up
    // to ~72 KB so narrow layers pack several offsets into one stage
    // default stage cap 72 KB; CTA pairs with 256-wide outputs default to 48 KB stages: a
    // deeper ring measured 2.7% faster on 256x256 (146 vs 150 us, tensor pipe 48.0% vs 46.5%
    // of elapsed, 51.4% vs 49.2% of active cycles; profiles/r2_wide_256_256_pair_stage48.txt),
    // while 192-wide pairs lose 16% with it (110.6 vs 95.0 us)
    const int64_t skb = option(SPC_OPT_CONV_STAGE_KB);
    const size_t stage_cap0 = (size_t)std::max<int64_t>(8, (p.cg == 2 && p.BN == 256 && skb == 72) ? 48 : skb) * 1024;
    // carve the ring for `slots` index blocks; false when it gets fewer than min_stages
    size_t ring_bytes = 0, header = 0;
    auto carve = [&](int slots, size_t stage_cap, int min_stages) {
        header = align_up(sizeof(ConvSmem), 128) + (size_t)slots * blk_bytes + (bulk_red ? RED_STAGE_BYTES : 0);
        if (header + 1024 + 8 * 1024 > TC_SMEM_BUDGET) return false;
        const size_t avail = TC_SMEM_BUDGET - 1024 - header;   // 1024: alignment slack of the dynamic smem base
        ring_bytes = 0;
        for (int g = 0; g < 2; ++g) {
            const int rows = g == 0 ? p.bm : TC_BM;
            ConvParams::Ring &R = p.ring[g];
            const uint32_t kb_bl = p.kb_b / p.cg;   // this CTA's share of a weight tile
            R.kb_a = (uint32_t)(rows * p.BK * 2);
            R.nkb = (int)std::max<size_t>(1, std::min<size_t>(8, stage_cap / (R.kb_a + kb_bl)));
            R.a_bytes = R.nkb * R.kb_a;
            R.b_bytes = R.nkb * kb_bl;
            R.stages = (int)std::min<size_t>(16, avail / (R.a_bytes + R.b_bytes));
            if (R.stages < min_stages) return false;
            ring_bytes = std::max(ring_bytes, (size_t)R.stages * (R.a_bytes + R.b_bytes));
        }
        p.blk_slots = slots;
        return true;
    };
    // two index blocks (the next tile's indices load while this tile gathers) whenever they
    // fit beside an unshrunk ring of >= 2 stages: large ones (K = 5 OS, 64 KB per 128-row
    // tile) only on narrow layers (C3 level 0, 16 -> 16: 52.8 -> 48.9 us); shrinking the
    // stages to make room loses (32 / 64 / 128 channels: +15% / +28% / +22%)
    const size_t blk_cap = (size_t)std::max<int64_t>(0, option(SPC_OPT_CONV_BLK_KB)) * 1024;
    bool ok = 2 * blk_bytes <= std::max<size_t>(blk_cap, 64 * 1024) && carve(2, stage_cap0, 2);
    if (!ok) ok = carve(1, stage_cap0, 2);
    if (!ok) return fail(SPC_ERR_UNSUPPORTED, "spc_conv_forward: tile does not fit shared memory");
    p.hdr_off = (uint32_t)align_up(ring_bytes, 128);
    p.red_off = bulk_red ? (uint32_t)(p.hdr_off + align_up(sizeof(ConvSmem), 128) + (size_t)p.blk_slots * blk_bytes) : 0u;
    const size_t smem = 1024 + p.hdr_off + header;
    static uint64_t configured = 0;   // bit d: smem attributes set on device d
    const int dev = current_device();
    if (!(configured >> dev & 1)) {
        void (*ks[])(ConvParams) = {k_conv_tc<16, 128, 1>, k_conv_tc<32, 128, 1>, k_conv_tc<64, 128, 1>,
                                    k_conv_tc<16, 256, 1>, k_conv_tc<32, 256, 1>, k_conv_tc<64, 256, 1>,
                                    k_conv_tc<16, 128, 2>, k_conv_tc<32, 128, 2>, k_conv_tc<64, 128, 2>,
                                    k_conv_tc<16, 128, 1, true>, k_conv_tc<32, 128, 1, true>,
                                    k_conv_tc<64, 128, 1, true>, k_conv_tc<16, 256, 1, true>,
                                    k_conv_tc<32, 256, 1, true>, k_conv_tc<64, 256, 1, true>};
        for (auto k : ks) SPC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_BUDGET));
        configured |= 1ull << dev;
    }
    // persistent: one CTA per SM (tile geometry and counts live on the device)
    const int64_t tiles_cap = mode == 0 ? ((p.n_out_cap + TC_BM - 1) / TC_BM) * p.n_ntiles *
                                              (p.split_ok ? std::max(1, p.k_dense / 2) : 1)
                                        : (int64_t)num_sms();
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles_cap, num_sms()));
    const int64_t cap = option(SPC_OPT_CONV_MAX_CTAS);   // SMs left to a concurrent stream
    if (cap > 0) {
        grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, cap));
        // the device-side tile heuristics (split-K parts, 128 / 256-row tiles) count the CTAs
        // that actually run: parts sized for 148 on a 140-CTA grid left a second wave
        // (C2 three in flight with the tail capped at 140: 1.352 vs 1.203 ms)
        p.num_sms = std::min(p.num_sms, grid);
    }
    if (p.cg == 2) grid = 2 * std::max(1, std::min(grid, num_sms()) / 2);   // whole CTA pairs
    p.trace = trace_next(std::string("k_conv_tc ") + (mode == 0 ? "os" : "ws") + (p.cg == 2 ? " pair" : "") +
                         " n_out=" + std::to_string(p.n_out_cap) + " c_in=" + std::to_string(p.n_chunks * p.BK) +
                         " c_out=" + std::to_string(p.n_ntiles * p.BN) + " k_dense=" + std::to_string(p.k_dense) +
                         " lists=" + std::to_string(p.n_lists));
    if (p.cg == 2) {
        void (*k)(ConvParams) = p.BK == 64 ? k_conv_tc<64, 128, 2> : p.BK == 32 ? k_conv_tc<32, 128, 2> : k_conv_tc<16, 128, 2>;
        SPC_CUDA(launch_pdl_cluster(k, dim3(grid), dim3(TC_THREADS), smem, st, 2, p));
        return SPC_OK;
    }
    // the fused BN / ReLU epilogue is a separate instantiation: its extra
    // epilogue registers cost the plain kernel 2% of a C2 step when compiled in (A/B)
    void (*k)(ConvParams);
    if (out_kind == OUT_FINAL && epi_on(p.epi))
        k = p.bm == 256 ? (p.BK == 64 ? k_conv_tc<64, 256, 1, true> : p.BK == 32 ? k_conv_tc<32, 256, 1, true>
                                                                              : k_conv_tc<16, 256, 1, true>)
                        : (p.BK == 64 ? k_conv_tc<64, 128, 1, true> : p.BK == 32 ? k_conv_tc<32, 128, 1, true>
                                                                              : k_conv_tc<16, 128, 1, true>);
    else
        k = p.bm == 256 ? (p.BK == 64 ? k_conv_tc<64, 256, 1> : p.BK == 32 ? k_conv_tc<32, 256, 1> : k_conv_tc<16, 256, 1>)
                        : (p.BK == 64 ? k_conv_tc<64, 128, 1> : p.BK == 32 ? k_conv_tc<32, 128, 1> : k_conv_tc<16, 128, 1>);
    SPC_CUDA(launch_pdl(k, dim3(grid), dim3(TC_THREADS), smem, st, p));
    return SPC_OK;
}

extern "C" spc_status spc_conv_forward(const spc_kmap *km, const void *f_in, int64_t ld_in, int32_t in_dtype,
                                       int32_t c_in, const void *weight, int32_t c_out, void *f_out, int64_t ld_out,
                                       int32_t out_dtype, const void *residual, int64_t ld_res, void *ws,
                                       size_t ws_bytes, void *stream) {
    return spc_conv_forward_ex(km, f_in, ld_in, in_dtype, c_in, weight, c_out, f_out, ld_out, out_dtype, residual,
                               ld_res, nullptr, ws, ws_bytes, stream);
}

extern "C" spc_status spc_conv_forward_ex(const spc_kmap *km, const void *f_in, int64_t ld_in, int32_t in_dtype,
                                          int32_t c_in, const void *weight, int32_t c_out, void *f_out,
                                          int64_t ld_out, int32_t out_dtype, const void *residual, int64_t ld_res,
                                          const spc_epilogue *epi, void *ws, size_t ws_bytes, void *stream) {
    SPC_CHECK_ARG(km && weight && f_out, "null pointer");
    SPC_CHECK_ARG(in_dtype >= SPC_F32 && in_dtype <= SPC_BF16 && out_dtype >= SPC_F32 && out_dtype <= SPC_BF16,
                  "bad dtype");
    SPC_CHECK_ARG(c_in > 0 && c_out > 0 && ld_in >= c_in && ld_out >= c_out, "bad channel counts / leading dims");
    SPC_CHECK_ARG(f_in || km->n_in == 0, "null f_in");
    SPC_CHECK_ARG(!residual || ld_res >= c_out, "bad ld_res");
    const size_t ein = elem_size(in_dtype), eout = elem_size(out_dtype);
    SPC_CHECK_ARG(((uintptr_t)f_in % 16) == 0 && (ld_in * ein) % 16 == 0, "f_in rows must be 16-byte aligned");
    SPC_CHECK_ARG(((uintptr_t)f_out % 16) == 0 && (ld_out * eout) % 16 == 0, "f_out rows must be 16-byte aligned");
    SPC_CHECK_ARG(!residual || (((uintptr_t)residual % 16) == 0 && (ld_res * eout) % 16 == 0),
                  "residual rows must be 16-byte aligned");
    cudaStream_t st = as_stream(stream);
    if (km->n_out == 0) return SPC_OK;
    const bool has_os = km->k_dense > 0, has_ws = km->n_lists > 0;

    ConvParams p;
    memset(&p, 0, sizeof(p));
    fill_map_params(p, km);
    p.f_in = static_cast<const char *>(f_in);
    p.ld_in_bytes = ld_in * (int64_t)ein;
    p.out_dtype = out_dtype;
    p.residual = residual;
    p.ld_res = ld_res;
    if (epi) p.epi = Epi{epi->scale, epi->shift, epi->relu};
    SPC_CHECK_ARG(!epi || ((uintptr_t)epi->scale % 16 == 0 && (uintptr_t)epi->shift % 16 == 0),
                  "epilogue scale / shift must be 16-byte aligned");

    // accumulator of the WS part (fp32)
    float *acc = nullptr;
    int64_t ld_acc = 0;
    if (has_ws) {
        if (out_dtype == SPC_F32 && !residual && !epi_on(p.epi)) {
            acc = static_cast<float *>(f_out);
            ld_acc = ld_out;
        } else {
            if (!ws || ws_bytes < spc_conv_workspace_size(km, c_out, out_dtype))
                return fail(SPC_ERR_WORKSPACE, "spc_conv_forward: ws too small");
            acc = static_cast<float *>(ws);
            ld_acc = c_out;
        }
    }

    if (in_dtype == SPC_F32) {
        SPC_CHECK_ARG(c_in % 4 == 0 && c_out % 8 == 0, "f32 path needs c_in % 4 == 0 and c_out % 8 == 0");
        const dim3 block(256);
        const unsigned gy = (unsigned)((c_out + SM_TN - 1) / SM_TN);
        if (has_os) {
            ConvParams q = p;
            q.mode = 0;
            q.out_kind = has_ws ? OUT_F32_STORE : OUT_FINAL;
            q.out = has_ws ? (void *)acc : f_out;
            q.ld_out = has_ws ? ld_acc : ld_out;
            SPC_CUDA(launch_pdl(k_conv_simt, dim3((unsigned)((km->n_out + SM_TM - 1) / SM_TM), gy), block, 0, st, q,
                                static_cast<const float *>(weight), (int)c_in, (int)c_out));
            SPC_LAUNCH_CHECK("k_conv_simt os");
        } else if (has_ws && acc == f_out) {
            SPC_CUDA(launch_pdl(k_zero_rows, dim3(1024), dim3(256), 0, st, acc, ld_acc, km->n_out, km->n_out_dev, (int)c_out));
        }
        if (has_ws) {
            ConvParams q = p;
            q.mode = 1;
            q.out_kind = OUT_F32_RED;
            q.out = acc;
            q.ld_out = ld_acc;
            const int64_t tiles_per = (km->n_out + SM_TM - 1) / SM_TM;
            SPC_CUDA(launch_pdl(k_conv_simt, dim3((unsigned)(tiles_per * 2 * km->n_lists), gy), block, 0, st, q,
                                static_cast<const float *>(weight), (int)c_in, (int)c_out));
            SPC_LAUNCH_CHECK("k_conv_simt ws");
            if (acc != f_out) {
                const int64_t work = km->n_out * (c_out / 8);
                SPC_CUDA(launch_pdl(k_convert, dim3((unsigned)std::min<int64_t>((work + 255) / 256, 8 * 148)), dim3(256), 0, st,
                    acc, ld_acc, km->n_out, km->n_out_dev, (int)c_out, (int)out_dtype, f_out, ld_out, residual, ld_res, 1, p.epi));
                SPC_LAUNCH_CHECK("k_convert");
            }
        }
        return SPC_OK;
    }

    // ---- tcgen05 path ------------------------------------------------------------------
    if (c_in % 16 || c_out % 16)
        return fail(SPC_ERR_UNSUPPORTED, "spc_conv_forward: f16/bf16 needs c_in and c_out multiples of 16");
    p.BK = pick_bk(c_in);
    p.BN = pick_bn(c_out);
    p.n_chunks = c_in / p.BK;
    p.n_ntiles = c_out / p.BN;
    p.tmem_cols = pow2_cols(p.BN);
    p.num_sms = num_sms();
    const int64_t force_tr = option(SPC_OPT_CONV_TILE_ROWS);
    p.force_tr = (force_tr == 128 || force_tr == 256) ? (int)force_tr : 0;
    p.split_min_unit = (int)std::max<int64_t>(1, option(SPC_OPT_CONV_SPLIT_MIN));
    p.claim_ahead = (int)std::max<int64_t>(1, std::min<int64_t>(3, option(SPC_OPT_CONV_CLAIM_AHEAD)));
    {   // weighted split when 2 * tiles <= this (default: the SM count)
        const int64_t st_opt = option(SPC_OPT_CONV_SPLIT_TILES);
        p.split_tiles_per_sm2 = st_opt > 0 ? (int)st_opt : p.num_sms;
    }
    // 256-row tiles (two MMAs per weight tile) whenever four accumulators fit TMEM; the
    // kernel drops to 128-row tiles on the device when the live row count is small
    p.bm = (4 * p.tmem_cols <= 512) ? 256 : 128;
    if (has_os && (size_t)BLK_SLOTS * p.bm * km->k_dense * 4 > 96 * 1024) p.bm = 128;   // OS index blocks (K=5)
    // CTA pairs (cta_group::2) for wide outputs, where a 128-row tile would re-read the whole
    // weight tile per 128 rows: a pair runs 256-row tiles with M = 256 MMAs, each CTA loading
    // half of every weight tile (half the L2 weight traffic per row, half the MMA issues).
    // Pairs walk their tiles statically and never split a tile's offsets, so an all-OS map
    // whose live size is unknown on the host (network maps) keeps single CTAs.
    {
        const int64_t pair_opt = option(SPC_OPT_CONV_CTA_PAIR);
        const bool wide = p.BN >= 192 && p.bm == 128 && (p.BN / 2) % 16 == 0;
        // measured: pairs win on large output-stationary launches (C5 256x256: 177 -> 169 us,
        // 192x192: 133 -> 116 us) and lose on the small weight-stationary levels of C2 (the
        // scatter epilogue dominates there and the pair hand-off adds latency)
        const bool big_os = has_os && !has_ws && !km->n_out_dev &&
                            ((km->n_out + 255) / 256) * p.n_ntiles >= p.num_sms / 2;
        p.cg = (pair_opt != 0 && wide && (big_os || pair_opt == 2) && !epi_on(p.epi)) ? 2 : 1;
    }
    p.tbufs = (p.bm == 256 ? 4 : 2) * p.tmem_cols <= 512 ? 2 : 1;
    p.kb_b = (uint32_t)(p.BN * p.BK * 2);
    p.idesc = ptx::umma_idesc_f16(in_dtype == SPC_BF16, TC_BM * p.cg, p.BN);
    p.wblob = static_cast<const char *>(weight);
    // workspace: fp32 accumulator + tile counters (zero on entry, zero on return)
    float *wacc = nullptr;
    int *wctr = nullptr;
    if (ws && ws_bytes >= spc_conv_workspace_size(km, c_out, out_dtype)) {
        wacc = static_cast<float *>(ws);
        wctr = reinterpret_cast<int *>(static_cast<char *>(ws) + align_up((size_t)km->n_out * c_out * 4, 256));
    }
    p.acc = wacc;
    p.ld_acc = c_out;
    p.tile_ctr = wctr;
    p.skip_list = -1;
    p.maps_ready = option(SPC_OPT_CONV_MAPS_READY) != 0 ? 1 : 0;
    // A11: identity maps need no gather.  A K = 1 submanifold layer is one dense TMA-fed
    // GEMM; with SPC_OPT_CONV_DENSE_CENTRE the centre of an all-weight-stationary
    // submanifold map (always matched, out_i += F_i W_centre) is computed the same
    // way and INITIALISES the fp32 accumulator, replacing its pair list and the zero fill
    // (off by default: on C2's small deep levels the extra launch costs more than the
    // centre list's scatter)
    // identity centre: one coordinate set in and out (not a range shard of one)
    const bool subm = km->geom.stride == 1 && !km->geom.transposed && km->in_keys == km->out_keys &&
                      km->n_in == km->n_out && km->n_in_dev == km->n_out_dev;
    if (subm && km->k_vol == 1 && km->k_dense == 1)
        return dense_forward(f_in, ld_in, in_dtype, c_in, weight, 0, c_out, p.BK, p.BN, km->n_out, km->n_out_dev, f_out,
                             ld_out, OUT_FINAL, out_dtype, residual, ld_res, p.epi, st);
    if (!has_ws) {
        // OS only: one launch; small levels split offsets over CTAs with the in-kernel fixup
        p.split_ok = (p.cg == 1 && wacc && km->k_dense >= 4 && option(SPC_OPT_CONV_OS_SPLIT) != 0) ? 1 : 0;
        return launch_tc(p, 0, OUT_FINAL, f_out, ld_out, st);
    }
    p.split_ok = 0;
    if (!acc) return fail(SPC_ERR_WORKSPACE, "spc_conv_forward: ws too small");
    const int centre = (km->k_vol - 1) / 2;
    // (the zero offset sits at the centre of a centred box only: every size odd)
    const spc_geom &gm = km->geom;
    const bool centred = gm.kernel_size % 2 == 1 && (gm.kernel_size_y <= 0 || gm.kernel_size_y % 2 == 1) &&
                         (gm.kernel_size_z <= 0 || gm.kernel_size_z % 2 == 1);
    if (!has_os && subm && centred && km->k_vol > 1 && option(SPC_OPT_CONV_DENSE_CENTRE) != 0)
        for (int l = 0; l < km->n_lists; ++l)
            if (km->list_k[l] == centre) p.skip_list = l;
    if (has_os) {
        spc_status s = launch_tc(p, 0, OUT_F32_STORE, acc, ld_acc, st);
        if (s != SPC_OK) return s;
    } else if (p.skip_list >= 0) {
        spc_status s = dense_forward(f_in, ld_in, in_dtype, c_in, weight, centre, c_out, p.BK, p.BN, km->n_out,
                                     km->n_out_dev, acc, ld_acc, OUT_F32_STORE, SPC_F32, nullptr, 0, Epi{}, st);
        if (s != SPC_OK) return s;
    } else if (acc == f_out) {
        SPC_CUDA(launch_pdl(k_zero_rows, dim3(1024), dim3(256), 0, st, acc, ld_acc, km->n_out, km->n_out_dev, (int)c_out));
        SPC_LAUNCH_CHECK("k_zero_rows");
    }
    {
        spc_status s = launch_tc(p, 1, OUT_F32_RED, acc, ld_acc, st);
        if (s != SPC_OK) return s;
    }
    if (acc != f_out) {
        const int64_t work = km->n_out * (c_out / 8);
        SPC_CUDA(launch_pdl(k_convert, dim3((unsigned)std::min<int64_t>((work + 255) / 256, 8 * 148)), dim3(256), 0, st,
            acc, ld_acc, km->n_out, km->n_out_dev, (int)c_out, (int)out_dtype, f_out, ld_out, residual, ld_res, 1, p.epi));
        SPC_LAUNCH_CHECK("k_convert");
    }
    return SPC_OK;
}

