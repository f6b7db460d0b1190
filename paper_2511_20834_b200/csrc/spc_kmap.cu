// spc_kmap.cu -- A4-A8: one-shot z-delta kernel-map build on packed keys (§5.2,
// P:341 packed queries, P:393-421 layouts and symmetric halving).
//
// CTA = tile of KM_BM sorted outputs.  For a fixed offset group the queries of a tile are
// sorted, so every match of (tile, group g) lies in ONE contiguous window of the sorted
// input keys: [lb(q_first + d_anchor(g)), lb(q_last + d_last(g) + 1)).  Phase A finds the
// 2*K^2 window bounds (parallel global lower_bounds), phase A' stages the windows in
// shared memory (coalesced), phase B runs the paper's z-delta search per (output, group)
// inside the window: one lower_bound for the anchor query, then a forward cursor for the
// other K-1 members.  Both layouts are written straight from phase B:
//   OS (dense offsets): staged as a [KM_BM x K_dense] int32 block in smem, flushed with
//       coalesced 16-byte stores (no transpose pass);
//   WS (sparse offsets): (in, out) pairs appended with one warp-aggregated atomicAdd per
//       (warp, offset) (no filter pass); halved for submanifold layers.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "spc_common.cuh"

namespace spc {

constexpr int KM_BM = 128;          // outputs per tile
constexpr int KM_THREADS = 256;
constexpr int KM_WIN_CAP = 4096;    // staged window keys per tile (32 KB)

// Compact per-map descriptor; the offset tables (packed query deltas, weight slots,
// dense columns, WS lists) are rebuilt in shared memory from it, so one launch can build
// every map of a network (phase 2 of network-wide indexing) with the descriptors
// passed as kernel parameters.
struct KmapDesc {
    const uint64_t *in;
    const uint64_t *out;
    int64_t n_in_cap, n_out_cap;
    const int64_t *n_in_dev;
    const int64_t *n_out_dev;
    int32_t *os;
    int2 *pairs;
    int32_t *counts;
    uint32_t *tile_mask;
    unsigned long long *stats;
    int64_t list_stride;
    int32_t spacing;
    int16_t K, k_dense, tile_words, t_eff;
    int8_t transposed, halved;
};

constexpr int KM_MAX_MAPS = 24;

struct KmapBatch {
    int n_maps;
    int bits_y, bits_z;
    unsigned int *work_ctr;   // zeroed before the launch
    KmapDesc d[KM_MAX_MAPS];
};

__device__ __forceinline__ int64_t lower_bound_g(const uint64_t *__restrict__ a, int64_t n, uint64_t q) {
    int64_t lo = 0, len = n;
    while (len > 0) {
        int64_t half = len >> 1;
        if (__ldg(a + lo + half) < q) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return lo;
}

__device__ __forceinline__ int lower_bound_s(const uint64_t *a, int n, uint64_t q) {
    int lo = 0, len = n;
    while (len > 0) {
        int half = len >> 1;
        if (a[lo + half] < q) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return lo;
}

// zero the per-map counters / stats and the work counter
__global__ void k_kmap_prep(const __grid_constant__ KmapBatch b) {
    const int m = blockIdx.x;
    if (m == 0 && threadIdx.x == 0) *b.work_ctr = 0;
    if (m >= b.n_maps) return;
    for (int i = threadIdx.x; i < 2 * SPC_MAX_KVOL; i += blockDim.x) b.d[m].counts[i] = 0;
    if (b.d[m].stats && threadIdx.x < 2) b.d[m].stats[threadIdx.x] = 0;
}

__global__ void __launch_bounds__(KM_THREADS) k_kmap_zdelta(const __grid_constant__ KmapBatch B) {
    extern __shared__ __align__(16) unsigned char km_smem[];
    __shared__ int64_t win_lo[25];
    __shared__ int win_len[25];
    __shared__ int win_base[25];    // -1: window not staged, use global search
    __shared__ uint32_t smask[4];   // tile bit mask over dense columns (<= 125)
    __shared__ int64_t s_delta[SPC_MAX_KVOL];
    __shared__ int16_t s_kslot[SPC_MAX_KVOL], s_dcol[SPC_MAX_KVOL], s_list[SPC_MAX_KVOL];
    __shared__ uint8_t s_need[25];
    __shared__ int s_prefix[KM_MAX_MAPS + 1];
    __shared__ int s_work, s_cur_map;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        int acc = 0;
        for (int m = 0; m < B.n_maps; ++m) {
            s_prefix[m] = acc;
            const int64_t n_out = dev_count(B.d[m].n_out_cap, B.d[m].n_out_dev);
            acc += (int)((n_out + KM_BM - 1) / KM_BM);
        }
        s_prefix[B.n_maps] = acc;
        s_cur_map = -1;
    }
    __syncthreads();
    const int total = s_prefix[B.n_maps];

    for (;;) {
        if (tid == 0) s_work = (int)atomicAdd(B.work_ctr, 1u);
        __syncthreads();
        const int v = s_work;
        if (v >= total) break;
        int m = 0;
        while (s_prefix[m + 1] <= v) ++m;
        const KmapDesc &p = B.d[m];
        const int tile = v - s_prefix[m];
        const int K = p.K, G = K * K, KD = p.k_dense, r = (K - 1) / 2, kv = K * K * K;
        // ---- per-map tables (rebuilt only when the map changes) -------------------------
        if (s_cur_map != m) {
            if (tid < kv) {
                const int g = tid / K, mm = tid % K;
                const int ex = g / K - r, ey = g % K - r;
                const int ez = p.transposed ? r - mm : mm - r;   // ascending query order
                const int k = ((ex + r) * K + (ey + r)) * K + (ez + r);
                int64_t d = (int64_t)ex * p.spacing * (1ll << (B.bits_y + B.bits_z)) +
                            (int64_t)ey * p.spacing * (1ll << B.bits_z) + (int64_t)ez * p.spacing;
                s_delta[tid] = p.transposed ? -d : d;
                s_kslot[tid] = (int16_t)k;
                // per weight offset k == tid: dense column / WS list (same rule as make_plan)
                const int kx = tid / (K * K) - r, ky = (tid / K) % K - r, kz = tid % K - r;
                const int centre = (kv - 1) / 2;
                int dcol = -1, lst = -1, nd = 0, nl = 0;
                for (int k2 = 0; k2 <= tid; ++k2) {
                    const int l1 = abs(k2 / (K * K) - r) + abs((k2 / K) % K - r) + abs(k2 % K - r);
                    const bool dense = l1 < p.t_eff;
                    const bool stored = !dense && (!p.halved || k2 <= centre);
                    if (k2 == tid) {
                        dcol = dense ? nd : -1;
                        lst = stored ? nl : -1;
                    }
                    nd += dense;
                    nl += stored;
                }
                (void)kx; (void)ky; (void)kz;
                s_dcol[tid] = (int16_t)dcol;
                s_list[tid] = (int16_t)lst;
            }
            __syncthreads();
            if (tid < G) {
                bool need = false;
                for (int mm = 0; mm < K; ++mm) {
                    const int k = s_kslot[tid * K + mm];
                    need |= s_dcol[k] >= 0 || s_list[k] >= 0;
                }
                s_need[tid] = need;
            }
            if (tid == 0) s_cur_map = m;
        }
        if (tid < 4) smask[tid] = 0;
        __syncthreads();

        const int64_t n_out = dev_count(p.n_out_cap, p.n_out_dev);
        const int64_t n_in = dev_count(p.n_in_cap, p.n_in_dev);
        const int64_t row0 = (int64_t)tile * KM_BM;
        const int rows = (int)imin64(KM_BM, n_out - row0);
        int32_t *os_tile = reinterpret_cast<int32_t *>(km_smem);
        uint64_t *win = reinterpret_cast<uint64_t *>(km_smem + KM_BM * KD * 4);   // KM_BM*4 = 512 B multiple

        // ---- phase A: window bounds of every (tile, group) ----------------------------
        const uint64_t q_first = p.out[row0];
        const uint64_t q_last = p.out[row0 + rows - 1];
        if (tid < 2 * G) {
            const int g = tid >> 1;
            if (s_need[g]) {
                const uint64_t q = (tid & 1) ? q_last + (uint64_t)s_delta[g * K + K - 1] + 1ull
                                             : q_first + (uint64_t)s_delta[g * K];
                const int64_t b = lower_bound_g(p.in, n_in, q);
                if (tid & 1) win_len[g] = (int)imin64(b, INT32_MAX);   // hi for now
                else win_lo[g] = b;
            }
        }
        __syncthreads();
        if (tid == 0) {
            int base = 0;
            for (int g = 0; g < G; ++g) {
                if (!s_need[g]) { win_base[g] = -1; win_len[g] = 0; continue; }
                int64_t len = (int64_t)win_len[g] - win_lo[g];
                if (len < 0) len = 0;
                win_len[g] = (int)len;
                if (base + len <= KM_WIN_CAP) { win_base[g] = base; base += (int)len; }
                else win_base[g] = -1;
            }
        }
        __syncthreads();
        // ---- phase A': stage windows (one warp per group, coalesced) -----------------------
        for (int g = warp; g < G; g += KM_THREADS / 32) {
            if (win_base[g] < 0) continue;
            const uint64_t *src = p.in + win_lo[g];
            uint64_t *dst = win + win_base[g];
            for (int e = lane; e < win_len[g]; e += 32) dst[e] = __ldg(src + e);
        }
        __syncthreads();

        // ---- phase B: z-delta search per (output, group) ---------------------------------
        unsigned long long n_search = 0, n_probe = 0;
        const int chunks = KM_BM / 32;
        for (int item = warp; item < G * chunks; item += KM_THREADS / 32) {
            const int g = item / chunks, ch = item - g * chunks;
            if (!s_need[g]) continue;
            const int lr = ch * 32 + lane;               // local row
            const bool valid = lr < rows;
            const int64_t i = row0 + lr;
            const uint64_t q = valid ? p.out[i] : 0;
            const bool staged = win_base[g] >= 0;
            const uint64_t *wk = staged ? win + win_base[g] : p.in + win_lo[g];
            const int wl = win_len[g];
            int pos = 0;
            if (valid) {
                pos = lower_bound_s(wk, wl, q + (uint64_t)s_delta[g * K]);
                ++n_search;
            }
            for (int mm = 0; mm < K; ++mm) {
                const uint64_t query = q + (uint64_t)s_delta[g * K + mm];
                bool match = false;
                if (valid) {
                    while (pos < wl && wk[pos] < query) { ++pos; ++n_probe; }
                    match = pos < wl && wk[pos] == query;
                }
                const int k = s_kslot[g * K + mm];
                const int32_t j = match ? (int32_t)(win_lo[g] + pos) : -1;
                const unsigned bal = __ballot_sync(0xffffffffu, match);
                if (lane == 0 && bal) atomicAdd(&p.counts[k], __popc(bal));
                const int col = s_dcol[k];
                if (col >= 0) {
                    if (valid) os_tile[lr * KD + col] = j;
                    if (lane == 0 && bal) atomicOr(&smask[col >> 5], 1u << (col & 31));
                } else {
                    const int l = s_list[k];
                    if (l >= 0 && bal) {
                        int base = 0;
                        if (lane == 0) base = atomicAdd(&p.counts[SPC_MAX_KVOL + l], __popc(bal));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (match) {
                            int2 pr = make_int2(j, (int32_t)i);
                            p.pairs[(int64_t)l * p.list_stride + base + __popc(bal & lanemask_lt())] = pr;
                        }
                    }
                }
            }
        }
        if (p.stats) {
            for (int o = 16; o > 0; o >>= 1) {
                n_search += __shfl_xor_sync(0xffffffffu, n_search, o);
                n_probe += __shfl_xor_sync(0xffffffffu, n_probe, o);
            }
            if (lane == 0) {
                atomicAdd(&p.stats[0], n_search);
                atomicAdd(&p.stats[1], n_probe);
            }
        }
        __syncthreads();
        // ---- phase C: flush the OS block (contiguous rows*KD int32) -----------------------
        if (KD > 0) {
            int32_t *dst = p.os + row0 * KD;
            const int totalv = rows * KD;
            const int nvec = totalv / 4;   // row0*KD*4 is 16-byte aligned (KM_BM = 128)
            int4 *d4 = reinterpret_cast<int4 *>(dst);
            const int4 *s4 = reinterpret_cast<const int4 *>(os_tile);
            for (int e = tid; e < nvec; e += KM_THREADS) d4[e] = s4[e];
            for (int e = nvec * 4 + tid; e < totalv; e += KM_THREADS) dst[e] = os_tile[e];
            if (tid < p.tile_words) p.tile_mask[(int64_t)tile * p.tile_words + tid] = smask[tid];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------
// density order of the OS part (SPC_KMAP_DENSITY_ORDER): outputs stably sorted by which
// offset directions they have neighbours in, so a 128-row tile of similar neighbour
// patterns has fewer non-empty offset chunks and fewer sentinel rows.  Any row order
// gives the same Eq. (2) result; this one only changes the work per tile.
// Key of an output: bit cls[c] set iff it matches at dense column c, where cls maps an
// offset and its mirror (k, K^3-1-k) to one bit (the centre of a submanifold map, always
// matched, to none), folded onto <= 16 bits.  All ordered maps of a build are sorted
// together: key = map tag above the mask bits, rows concatenated by live counts.
// ------------------------------------------------------------------------------------
constexpr int ORD_MAX = 8;
struct OrderJob {
    const int32_t *os;
    int32_t *os_ord;
    uint32_t *mask_ord;
    int32_t *rows;
    const int64_t *n_dev;
    int64_t n_cap;
    int64_t tile0;            // first permute CTA of this map
    int k_dense, words;
    int8_t cls[SPC_MAX_KVOL];
};
struct OrderBatch {
    int n_jobs, key_bits;
    int64_t *total_dev;       // sum of live rows (written by k_ord_keys)
    uint64_t *keys;
    OrderJob j[ORD_MAX];
};

__device__ __forceinline__ int64_t ord_base(const OrderBatch &B, int job, int64_t &n_job) {
    int64_t base = 0;
    for (int q = 0; q < job; ++q) base += dev_count(B.j[q].n_cap, B.j[q].n_dev);
    n_job = dev_count(B.j[job].n_cap, B.j[job].n_dev);
    return base;
}

__global__ void k_ord_keys(const __grid_constant__ OrderBatch B) {
    int64_t base = 0;
    for (int q = 0; q < B.n_jobs; ++q) {
        const OrderJob &J = B.j[q];
        const int64_t n = dev_count(J.n_cap, J.n_dev);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
            const int32_t *row = J.os + i * J.k_dense;
            uint32_t m = 0;
            for (int c = 0; c < J.k_dense; ++c)
                if (J.cls[c] >= 0 && row[c] >= 0) m |= 1u << J.cls[c];
            B.keys[base + i] = ((uint64_t)q << B.key_bits) | m;
        }
        base += n;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *B.total_dev = base;
}

// one CTA per 128-row tile of one map: row p of the ordered table = row rows[p] of the
// canonical one (warp-cooperative row copies), tile mask words by warp ballots
__global__ void __launch_bounds__(128) k_ord_permute(const __grid_constant__ OrderBatch B,
                                                     const int32_t *__restrict__ sorted_pos) {
    __shared__ int32_t src_s[128];
    __shared__ uint32_t wm[4][4];
    int job = 0;
    while (job + 1 < B.n_jobs && B.j[job + 1].tile0 <= blockIdx.x) ++job;
    const OrderJob &J = B.j[job];
    int64_t n;
    const int64_t base = ord_base(B, job, n);
    const int64_t p0 = (int64_t)(blockIdx.x - J.tile0) * 128;
    if (p0 >= n) return;
    const int64_t p = p0 + threadIdx.x;
    int32_t src = -1;
    if (p < n) {
        src = (int32_t)(sorted_pos[base + p] - base);
        J.rows[p] = src;
    }
    src_s[threadIdx.x] = src;
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t m[4] = {0u, 0u, 0u, 0u};
    for (int i = 0; i < 32; ++i) {
        const int r = w * 32 + i;
        const int32_t sr = src_s[r];
        if (sr < 0) break;
        const int32_t *srow = J.os + (int64_t)sr * J.k_dense;
        int32_t *drow = J.os_ord + (p0 + r) * J.k_dense;
        for (int c0 = 0, q = 0; c0 < J.k_dense; c0 += 32, ++q) {
            const int c = c0 + lane;
            int32_t v = -1;
            if (c < J.k_dense) {
                v = srow[c];
                drow[c] = v;
            }
            m[q & 3] |= __ballot_sync(0xffffffffu, v >= 0);
        }
    }
    if (lane == 0)
        for (int q = 0; q < 4; ++q) wm[w][q] = m[q];
    __syncthreads();
    if (threadIdx.x < J.words) {
        const int q = threadIdx.x;
        J.mask_ord[(p0 / 128) * J.words + q] = wm[0][q] | wm[1][q] | wm[2][q] | wm[3][q];
    }
}

// scratch of one grouped order over `rows_cap` concatenated rows
static size_t order_scratch_bytes(int64_t rows_cap) {
    Sizer z;
    z.take<int64_t>(4);
    z.take<uint64_t>((size_t)rows_cap);   // keys
    z.take<uint64_t>((size_t)rows_cap);   // sorted keys
    z.take<int32_t>((size_t)rows_cap);    // sorted positions
    return z.used + radix_sort_workspace(rows_cap, true) + 512;
}

static spc_status run_orders(const std::vector<OrderJob> &jobs, void *scratch, size_t scratch_bytes, cudaStream_t st) {
    for (size_t j0 = 0; j0 < jobs.size(); j0 += ORD_MAX) {
        OrderBatch B;
        memset(&B, 0, sizeof(B));
        B.n_jobs = (int)std::min<size_t>(ORD_MAX, jobs.size() - j0);
        int64_t cap = 0, tiles = 0;
        int bits = 1;
        for (int q = 0; q < B.n_jobs; ++q) {
            B.j[q] = jobs[j0 + q];
            B.j[q].tile0 = tiles;
            tiles += (B.j[q].n_cap + 127) / 128;
            cap += B.j[q].n_cap;
            for (int c = 0; c < B.j[q].k_dense; ++c) bits = std::max(bits, (int)B.j[q].cls[c] + 1);
        }
        if (cap == 0) continue;
        int tag_bits = 0;
        while ((1 << tag_bits) < B.n_jobs) ++tag_bits;
        B.key_bits = bits;
        Bump b(scratch, scratch_bytes);
        B.total_dev = b.take<int64_t>(4);
        B.keys = b.take<uint64_t>((size_t)cap);
        uint64_t *keys_sorted = b.take<uint64_t>((size_t)cap);
        int32_t *pos = b.take<int32_t>((size_t)cap);
        const size_t rws = radix_sort_workspace(cap, true);
        void *rw = b.take<uint8_t>(rws);
        if (!b.ok()) return fail(SPC_ERR_WORKSPACE, "kernel-map density order: scratch too small");
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((cap + 255) / 256, 4 * (int64_t)num_sms()));
        k_ord_keys<<<grid, 256, 0, st>>>(B);
        SPC_LAUNCH_CHECK("k_ord_keys");
        spc_status s = radix_sort(B.keys, nullptr, cap, B.total_dev, bits + tag_bits, keys_sorted, pos, rw, rws, st,
                                  false);
        if (s != SPC_OK) return s;
        k_ord_permute<<<(unsigned)tiles, 128, 0, st>>>(B, pos);
        SPC_LAUNCH_CHECK("k_ord_permute");
    }
    return SPC_OK;
}

// ------------------------------------------------------------------------------------
// host: plan (offset tables, dense/sparse split, lists) and entry points
// ------------------------------------------------------------------------------------
struct KmapPlan {
    int K = 0, r = 0, k_vol = 0, k_dense = 0, n_lists = 0, halved = 0, t_eff = 0, spacing = 1, centre_col = -1;
    int16_t dense_k[SPC_MAX_KVOL], list_k[SPC_MAX_KVOL];
    int8_t list_mirror[SPC_MAX_KVOL];
    int16_t dense_col[SPC_MAX_KVOL], list_id[SPC_MAX_KVOL];
    int8_t ord_cls[SPC_MAX_KVOL];   // density-order key bit of each dense column (-1: none)
    uint8_t group_needed[25];
};

static spc_status make_plan(const spc_geom &g, int32_t t, uint32_t flags, KmapPlan &pl) {
    if (g.kernel_size < 1 || g.kernel_size % 2 == 0 || g.kernel_size > 5)
        return fail(SPC_ERR_UNSUPPORTED, "kernel_size must be odd and <= 5 (P:111), got " +
                                             std::to_string(g.kernel_size));
    if (g.stride < 1 || g.dilation < 1 || g.tensor_stride < 1)
        return fail(SPC_ERR_INVALID_ARG, "stride, dilation and tensor_stride must be >= 1");
    if (g.transposed && g.stride == 1)
        return fail(SPC_ERR_INVALID_ARG, "a transposed map needs stride > 1");
    pl.K = g.kernel_size;
    pl.r = (pl.K - 1) / 2;
    pl.k_vol = pl.K * pl.K * pl.K;
    pl.spacing = g.tensor_stride * g.dilation;
    const int l1max = 3 * pl.r;
    pl.t_eff = (t < 0 || t > l1max + 1) ? l1max + 1 : t;
    const bool subm = g.stride == 1 && !g.transposed;
    pl.halved = (flags & SPC_KMAP_HALVE_SYMMETRIC) && subm ? 1 : 0;
    const int centre = (pl.k_vol - 1) / 2;
    pl.k_dense = pl.n_lists = 0;
    pl.centre_col = -1;
    for (int k = 0; k < pl.k_vol; ++k) {
        int ex = k / (pl.K * pl.K) - pl.r, ey = (k / pl.K) % pl.K - pl.r, ez = k % pl.K - pl.r;
        int l1 = abs(ex) + abs(ey) + abs(ez);
        pl.dense_col[k] = -1;
        pl.list_id[k] = -1;
        if (l1 < pl.t_eff) {
            if (subm && k == centre) pl.centre_col = pl.k_dense;   // always matched
            pl.dense_col[k] = (int16_t)pl.k_dense;
            pl.dense_k[pl.k_dense++] = (int16_t)k;
        } else if (!pl.halved || k <= centre) {
            pl.list_id[k] = (int16_t)pl.n_lists;
            pl.list_mirror[pl.n_lists] = (pl.halved && k < centre) ? 1 : 0;
            pl.list_k[pl.n_lists++] = (int16_t)k;
        }
    }
    // density-order key: an offset and its mirror share a bit; the centre of a
    // submanifold map (always matched) has none; <= 16 bits (classes folded)
    {
        int rank[SPC_MAX_KVOL];
        for (int k = 0; k < pl.k_vol; ++k) rank[k] = -1;
        int ncls = 0;
        for (int k = 0; k < pl.k_vol; ++k) {   // ascending pair index min(k, mirror)
            const int m = pl.k_vol - 1 - k;
            if (k > m) continue;
            const bool used = pl.dense_col[k] >= 0 || pl.dense_col[m] >= 0;
            if (!used || (subm && k == centre)) continue;
            rank[k] = rank[m] = ncls++;
        }
        for (int c = 0; c < pl.k_dense; ++c) {
            const int r = rank[pl.dense_k[c]];
            pl.ord_cls[c] = (int8_t)(r < 0 ? -1 : r % 16);
        }
    }
    for (int gi = 0; gi < pl.K * pl.K; ++gi) {
        bool need = false;
        for (int m = 0; m < pl.K; ++m) {
            int k = gi * pl.K + m;
            need |= pl.dense_col[k] >= 0 || pl.list_id[k] >= 0;
        }
        pl.group_needed[gi] = need;
    }
    return SPC_OK;
}

struct KmapLayout {
    size_t os, pairs, counts, mask, stats, total;
    size_t rows, os_ord, mask_ord, scratch, scratch_bytes;   // density order
    int64_t tiles;
    int words;
};

static bool wants_order(const KmapPlan &pl, uint32_t flags) { return (flags & SPC_KMAP_DENSITY_ORDER) && pl.k_dense >= 2; }

// scratch: include the density-order sort scratch (standalone builds; a network build
// sorts all its maps together in scratch of its own)
static KmapLayout layout_of(const KmapPlan &pl, int64_t n_out, uint32_t flags, bool scratch = true) {
    KmapLayout L{};
    L.tiles = (n_out + KM_BM - 1) / KM_BM;
    L.words = (pl.k_dense + 31) / 32;
    size_t off = 0;
    auto take = [&](size_t bytes) { off = align_up(off, 256); size_t at = off; off += bytes; return at; };
    L.os = take(sizeof(int32_t) * (size_t)n_out * pl.k_dense);
    L.pairs = take(sizeof(int2) * (size_t)n_out * pl.n_lists);
    L.counts = take(sizeof(int32_t) * 2 * SPC_MAX_KVOL);
    L.mask = take(sizeof(uint32_t) * (size_t)(L.tiles * L.words));
    L.stats = take(sizeof(unsigned long long) * 2 + 64);   // + a launch work counter
    if (wants_order(pl, flags)) {
        L.rows = take(sizeof(int32_t) * (size_t)n_out);
        L.os_ord = take(sizeof(int32_t) * (size_t)n_out * pl.k_dense);
        L.mask_ord = take(sizeof(uint32_t) * (size_t)(L.tiles * L.words));
        if (scratch) {
            L.scratch_bytes = order_scratch_bytes(n_out);
            L.scratch = take(L.scratch_bytes);
        }
    }
    L.total = align_up(off, 256);
    return L;
}


size_t kmap_smem_bytes(int k_dense) { return (size_t)KM_BM * k_dense * 4 + (size_t)KM_WIN_CAP * 8; }

struct DeferState {
    bool active = false;
    KmapBatch b;
    int max_kd = 0;
    int64_t tiles = 0;
    std::vector<OrderJob> orders;
    void *scratch = nullptr;   // density-order scratch of the batch
    size_t scratch_bytes = 0;
};
static thread_local DeferState g_defer;

static void fill_desc(KmapDesc &d, const spc_kmap &km, const KmapPlan &pl) {
    memset(&d, 0, sizeof(d));
    d.in = km.in_keys;
    d.out = km.out_keys;
    d.n_in_cap = km.n_in;
    d.n_out_cap = km.n_out;
    d.n_in_dev = km.n_in_dev;
    d.n_out_dev = km.n_out_dev;
    d.os = km.os_table;
    d.pairs = reinterpret_cast<int2 *>(km.ws_pairs);
    d.counts = km.counts_dev;
    d.tile_mask = km.tile_mask_dev;
    d.stats = km.search_stats_dev;
    d.list_stride = km.n_out;
    d.spacing = pl.spacing;
    d.K = (int16_t)pl.K;
    d.k_dense = (int16_t)pl.k_dense;
    d.tile_words = (int16_t)km.tile_words;
    d.t_eff = (int16_t)pl.t_eff;
    d.transposed = (int8_t)km.geom.transposed;
    d.halved = (int8_t)pl.halved;
}

static spc_status launch_kmaps(const KmapBatch &b, int max_k_dense, int64_t max_tiles, cudaStream_t st) {
    static int configured = 0;
    if (!configured) {
        SPC_CUDA(cudaFuncSetAttribute(k_kmap_zdelta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kmap_smem_bytes(SPC_MAX_KVOL)));
        configured = 1;
    }
    k_kmap_prep<<<b.n_maps > 0 ? b.n_maps : 1, 256, 0, st>>>(b);
    SPC_LAUNCH_CHECK("k_kmap_prep");
    const size_t smem = kmap_smem_bytes(max_k_dense);
    int per_sm = (int)((228 * 1024) / (smem + 4096));
    if (per_sm < 1) per_sm = 1;
    if (per_sm > 8) per_sm = 8;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(max_tiles, (int64_t)num_sms() * per_sm));
    k_kmap_zdelta<<<(unsigned)grid, KM_THREADS, smem, st>>>(b);
    SPC_LAUNCH_CHECK("k_kmap_zdelta");
    return SPC_OK;
}

}  // namespace spc

using namespace spc;

extern "C" size_t spc_kmap_bytes(spc_geom geom, int32_t t, uint32_t flags, int64_t n_in, int64_t n_out) {
    KmapPlan pl;
    if (make_plan(geom, t, flags, pl) != SPC_OK || n_out < 0) return 0;
    (void)n_in;
    return layout_of(pl, n_out, flags).total;
}

namespace spc {
__global__ void k_flag_dups(const uint64_t *keys, int64_t n_cap, const int64_t *n_dev, uint32_t *status,
                            uint32_t flag);
}

extern "C" spc_status spc_build_kmap(const uint64_t *in_keys, int64_t n_in, const int64_t *n_in_dev,
                                     const uint64_t *out_keys, int64_t n_out, const int64_t *n_out_dev,
                                     spc_pack_spec spec, spc_geom geom, int32_t t, uint32_t flags, void *buf,
                                     size_t buf_bytes, uint32_t *status, spc_kmap *kmap_out, void *stream) {
    SPC_CHECK_ARG(kmap_out, "null kmap_out");
    SPC_CHECK_ARG(n_in >= 0 && n_out >= 0, "negative size");
    SPC_CHECK_ARG(n_in < INT32_MAX && n_out < INT32_MAX, "sizes must fit int32 indices");
    SPC_CHECK_ARG((in_keys || n_in == 0) && (out_keys || n_out == 0), "null keys");
    KmapPlan pl;
    spc_status s = make_plan(geom, t, flags, pl);
    if (s != SPC_OK) return s;
    const KmapLayout L = layout_of(pl, n_out, flags, !g_defer.active);
    SPC_CHECK_ARG(buf && ((uintptr_t)buf % 256) == 0, "buf must be non-null and 256-byte aligned");
    if (buf_bytes < L.total) return fail(SPC_ERR_WORKSPACE, "spc_build_kmap: buffer too small");
    // reach check (reading A4): the planner guarantees headroom; here we only refuse
    // offsets that cannot be represented in the z field at all
    const int reach = pl.r * pl.spacing;
    if (reach >= (1 << (spec.bits_z - 1)) || reach >= (1 << (spec.bits_y - 1)) || reach >= (1 << (spec.bits_x - 1)))
        return fail(SPC_ERR_RANGE, "spc_build_kmap: kernel reach " + std::to_string(reach) +
                                       " does not fit the key fields");
    cudaStream_t st = as_stream(stream);
    char *base = static_cast<char *>(buf);

    spc_kmap &km = *kmap_out;
    memset(&km, 0, sizeof(km));
    km.geom = geom;
    km.t = pl.t_eff;
    km.k_vol = pl.k_vol;
    km.k_dense = pl.k_dense;
    km.n_lists = pl.n_lists;
    km.halved = pl.halved;
    km.tile_words = L.words;
    km.n_in = n_in;
    km.n_out = n_out;
    km.n_in_dev = n_in_dev;
    km.n_out_dev = n_out_dev;
    km.in_keys = in_keys;
    km.out_keys = out_keys;
    km.os_table = reinterpret_cast<int32_t *>(base + L.os);
    km.ws_pairs = reinterpret_cast<int32_t *>(base + L.pairs);
    km.counts_dev = reinterpret_cast<int32_t *>(base + L.counts);
    km.tile_mask_dev = reinterpret_cast<uint32_t *>(base + L.mask);
    km.search_stats_dev = (flags & SPC_KMAP_COUNT_SEARCHES) ? reinterpret_cast<unsigned long long *>(base + L.stats)
                                                             : nullptr;
    for (int c = 0; c < pl.k_dense; ++c) km.dense_k[c] = pl.dense_k[c];
    for (int l = 0; l < pl.n_lists; ++l) {
        km.list_k[l] = pl.list_k[l];
        km.list_mirror[l] = pl.list_mirror[l];
    }
    OrderJob job;
    memset(&job, 0, sizeof(job));
    const bool order = wants_order(pl, flags) && n_out > 0;
    if (order) {
        km.os_rows = reinterpret_cast<int32_t *>(base + L.rows);
        km.os_table_ord = reinterpret_cast<int32_t *>(base + L.os_ord);
        km.tile_mask_ord = reinterpret_cast<uint32_t *>(base + L.mask_ord);
        job.os = km.os_table;
        job.os_ord = km.os_table_ord;
        job.mask_ord = km.tile_mask_ord;
        job.rows = km.os_rows;
        job.n_dev = n_out_dev;
        job.n_cap = n_out;
        job.k_dense = pl.k_dense;
        job.words = L.words;
        for (int c = 0; c < pl.k_dense; ++c) job.cls[c] = pl.ord_cls[c];
    }
    if (n_out == 0) {
        SPC_CUDA(cudaMemsetAsync(base + L.counts, 0, L.stats + 2 * sizeof(unsigned long long) - L.counts, st));
        return SPC_OK;
    }
    if ((flags & SPC_KMAP_CHECK_SORTED) && status) {
        k_flag_dups<<<64, 256, 0, st>>>(in_keys, n_in, n_in_dev, status, SPC_FLAG_UNSORTED);
        k_flag_dups<<<64, 256, 0, st>>>(out_keys, n_out, n_out_dev, status, SPC_FLAG_UNSORTED);
    }

    if (g_defer.active) {
        // network-wide phase 2: collect, launch once in kmap_defer_end()
        KmapBatch &b = g_defer.b;
        if (b.n_maps >= KM_MAX_MAPS) return fail(SPC_ERR_CAPACITY, "too many distinct kernel maps in one batch");
        if (b.n_maps == 0) {
            b.bits_y = spec.bits_y;
            b.bits_z = spec.bits_z;
            b.work_ctr = reinterpret_cast<unsigned int *>(base + L.stats) + 4;
        } else if (b.bits_y != spec.bits_y || b.bits_z != spec.bits_z) {
            return fail(SPC_ERR_INVALID_ARG, "batched kernel maps must share one pack spec");
        }
        fill_desc(b.d[b.n_maps++], km, pl);
        g_defer.max_kd = std::max(g_defer.max_kd, pl.k_dense);
        g_defer.tiles += (int64_t)L.tiles;
        if (order) g_defer.orders.push_back(job);
        return SPC_OK;
    }
    KmapBatch b;
    memset(&b, 0, sizeof(b));
    b.n_maps = 1;
    b.bits_y = spec.bits_y;
    b.bits_z = spec.bits_z;
    b.work_ctr = reinterpret_cast<unsigned int *>(base + L.stats) + 4;   // scratch after the stats
    fill_desc(b.d[0], km, pl);
    s = launch_kmaps(b, pl.k_dense, (int64_t)L.tiles, st);
    if (s == SPC_OK && order) s = run_orders(std::vector<OrderJob>{job}, base + L.scratch, L.scratch_bytes, st);
    return s;
}

namespace spc {
void kmap_defer_begin(void *order_scratch, size_t order_scratch_bytes) {
    memset(&g_defer.b, 0, sizeof(g_defer.b));
    g_defer.max_kd = 0;
    g_defer.tiles = 0;
    g_defer.orders.clear();
    g_defer.scratch = order_scratch;
    g_defer.scratch_bytes = order_scratch_bytes;
    g_defer.active = true;
}
size_t kmap_bytes_batched(spc_geom geom, int32_t t, uint32_t flags, int64_t n_out) {
    KmapPlan pl;
    if (make_plan(geom, t, flags, pl) != SPC_OK || n_out < 0) return 0;
    return layout_of(pl, n_out, flags, false).total;
}
size_t kmap_order_rows(spc_geom geom, int32_t t, uint32_t flags, int64_t n_out) {
    KmapPlan pl;
    if (make_plan(geom, t, flags, pl) != SPC_OK) return 0;
    return wants_order(pl, flags) ? (size_t)n_out : 0;
}
size_t kmap_order_scratch_bytes(int64_t rows) { return rows > 0 ? order_scratch_bytes(rows) : 0; }
void kmap_defer_abort() { g_defer.active = false; }
spc_status kmap_defer_end(cudaStream_t st) {
    g_defer.active = false;
    if (g_defer.b.n_maps == 0) return SPC_OK;
    spc_status s = launch_kmaps(g_defer.b, g_defer.max_kd, g_defer.tiles, st);
    if (s == SPC_OK && !g_defer.orders.empty()) s = run_orders(g_defer.orders, g_defer.scratch, g_defer.scratch_bytes, st);
    return s;
}
}  // namespace spc

extern "C" spc_status spc_kmap_export(const spc_kmap *km, int32_t *triples_host, int64_t cap, int64_t *nnz_host,
                                      void *stream) {
    SPC_CHECK_ARG(km && nnz_host, "null pointer");
    cudaStream_t st = as_stream(stream);
    SPC_CUDA(cudaStreamSynchronize(st));
    int64_t n_out = km->n_out;
    if (km->n_out_dev) {
        int64_t v;
        SPC_CUDA(cudaMemcpy(&v, km->n_out_dev, sizeof(v), cudaMemcpyDeviceToHost));
        n_out = std::min(v, n_out);
    }
    std::vector<int32_t> counts(2 * SPC_MAX_KVOL);
    SPC_CUDA(cudaMemcpy(counts.data(), km->counts_dev, counts.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<int32_t> os((size_t)n_out * km->k_dense);
    if (!os.empty()) SPC_CUDA(cudaMemcpy(os.data(), km->os_table, os.size() * 4, cudaMemcpyDeviceToHost));
    struct Tr { int32_t k, i, j; };
    std::vector<Tr> tr;
    for (int64_t i = 0; i < n_out; ++i)
        for (int c = 0; c < km->k_dense; ++c) {
            int32_t j = os[(size_t)i * km->k_dense + c];
            if (j >= 0) tr.push_back({km->dense_k[c], (int32_t)i, j});
        }
    for (int l = 0; l < km->n_lists; ++l) {
        int32_t cnt = counts[SPC_MAX_KVOL + l];
        std::vector<int32_t> pr((size_t)cnt * 2);
        if (cnt) SPC_CUDA(cudaMemcpy(pr.data(), km->ws_pairs + (size_t)l * km->n_out * 2, pr.size() * 4,
                                     cudaMemcpyDeviceToHost));
        const int k = km->list_k[l];
        for (int32_t q = 0; q < cnt; ++q) {
            tr.push_back({k, pr[2 * q + 1], pr[2 * q]});
            if (km->list_mirror[l]) tr.push_back({km->k_vol - 1 - k, pr[2 * q], pr[2 * q + 1]});
        }
    }
    std::sort(tr.begin(), tr.end(), [](const Tr &a, const Tr &b) {
        if (a.k != b.k) return a.k < b.k;
        if (a.i != b.i) return a.i < b.i;
        return a.j < b.j;
    });
    *nnz_host = (int64_t)tr.size();
    if (triples_host)
        for (int64_t q = 0; q < (int64_t)tr.size() && q < cap; ++q) {
            triples_host[3 * q] = tr[q].k;
            triples_host[3 * q + 1] = tr[q].i;
            triples_host[3 * q + 2] = tr[q].j;
        }
    return SPC_OK;
}
