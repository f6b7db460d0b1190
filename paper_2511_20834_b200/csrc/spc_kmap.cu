// spc_kmap.cu -- A4-A8: one-shot z-delta kernel-map build on packed keys (§5.2,
// P:341 packed queries, P:393-421 layouts and symmetric halving).
//
// Outputs are cut into tiles of KM_BM sorted keys.  For a fixed offset group g (the K
// offsets sharing (dx, dy)) the queries of a tile are sorted, so every match of (tile, g)
// lies in ONE contiguous window of the sorted input keys:
// [lb(q_first + d_anchor(g)), lb(q_last + d_last(g) + 1)).
//   k_kmap_bounds: every window bound of every (map, tile, group) in one parallel pass.
//   k_kmap_zdelta: one CTA per (map, tile): the tile's K^2 windows staged in one shared
//       pool (coalesced), then the paper's z-delta search per output: one lower_bound for
//       the anchor query, then a forward cursor for the other K-1 members, one
//       warp per (group, 32-output chunk).  Both layouts are assembled in shared memory and
//       leave as contiguous streams: the OS block of the [n_out x K_dense] table (every
//       entry written once, -1 for no match: no transpose pass); each WS list's
//       (in, out) pairs compacted with one warp-aggregated reservation per (tile, list) (no
//       filter pass), halved for submanifold layers.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "spc_common.cuh"

namespace spc {

constexpr int KM_BM = 128;          // outputs per tile
constexpr int KM_THREADS = 256;
constexpr int KM_WARPS = KM_THREADS / 32;

// Compact per-map descriptor; the offset tables (packed query deltas, weight slots,
// dense columns, WS lists) are rebuilt in shared memory from it, so one launch can build
// every map of a network (phase 2 of network-wide indexing) with the descriptors
// passed as kernel parameters.
struct KmapDesc {
    const void *in;           // sorted keys: uint64 (KmapBatch.key_bytes 8) or uint32 (4)
    const void *out;
    int64_t n_in_cap, n_out_cap;
    const int64_t *n_in_dev;
    const int64_t *n_out_dev;
    int32_t *os;
    int2 *pairs;
    int32_t *counts;
    uint32_t *tile_mask;
    unsigned long long *stats;
    int32_t *bounds;          // [tiles][Kx*Ky][2] window bounds (k_kmap_bounds)
    int64_t list_stride;
    int32_t spacing;
    int32_t k_dense, tile_words, t_eff;   // (scalars int32: see kx below)
    // offset box: Kx x Ky groups of Kz members along z; per axis the
    // offsets e = lo .. lo + K - 1 (odd K centred as in Delta(K, s_p); even K from 0)
    // (int32: byte-wide fields cost 7% of the build -- sign-extending dynamic param loads)
    int32_t kx, ky, kz, lox, loy, loz;
    int32_t transposed, halved;
    int32_t ord_idx;                // density order: index among the ordered maps (-1: none)
    int8_t ord_cls[SPC_MAX_KVOL];   // density-order key bit of each dense column (-1: none)
    int8_t dcol[SPC_MAX_KVOL];      // weight offset -> dense column (-1: not dense)
    int8_t lst[SPC_MAX_KVOL];       // weight offset -> stored WS list (-1: none)
};

constexpr int KM_MAX_MAPS = 24;

struct KmapBatch {
    int n_maps;
    int bits_y, bits_z;
    unsigned int *work_ctr;   // zeroed before the launch
    int pool_keys;            // usable keys of the shared window pool (<= KM_POOL; SPC_OPT_KMAP_POOL_KEYS)
    int key_bytes;            // 8: 64-bit keys, 4: 32-bit single-scan keys
    // density order: keys of all ordered maps, concatenated in ord_idx order by live counts
    uint64_t *ord_keys;
    int64_t *ord_total;       // sum of their live rows (written by k_kmap_prep)
    int ord_key_bits;         // bit of the map tag (direction mask below, then the weight field)
    KmapDesc d[KM_MAX_MAPS];
};

template <typename KeyT>
__device__ __forceinline__ int64_t lower_bound_g(const KeyT *__restrict__ a, int64_t n, KeyT q) {
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
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    const int m = blockIdx.x;
    if (m == 0 && threadIdx.x == 0) {
        *b.work_ctr = 0;
        if (b.ord_total) {
            int64_t tot = 0;
            for (int q = 0; q < b.n_maps; ++q)
                if (b.d[q].ord_idx >= 0) tot += dev_count(b.d[q].n_out_cap, b.d[q].n_out_dev);
            *b.ord_total = tot;
        }
    }
    if (m >= b.n_maps) return;
    for (int i = threadIdx.x; i < 2 * SPC_MAX_KVOL; i += blockDim.x) b.d[m].counts[i] = 0;
    if (b.d[m].stats && threadIdx.x < 2) b.d[m].stats[threadIdx.x] = 0;
}

// packed query delta of member mm (ascending query order) of offset group g
__device__ __forceinline__ int64_t group_delta(const KmapDesc &p, int by, int bz, int g, int mm) {
    const int ex = g / p.ky + p.lox, ey = g % p.ky + p.loy;
    const int ez = p.transposed ? p.loz + p.kz - 1 - mm : p.loz + mm;
    const int64_t d = (int64_t)ex * p.spacing * (1ll << (by + bz)) + (int64_t)ey * p.spacing * (1ll << bz) +
                      (int64_t)ez * p.spacing;
    return p.transposed ? -d : d;
}

// phase A of every (map, tile, group) at once: the window [lo, hi) of the sorted input
// keys holding all matches of a tile's outputs for one offset group.  One thread per
// bound, so the global binary searches' latency chains all run concurrently instead of
// once per tile inside the build kernel.
template <typename KeyT>
__global__ void __launch_bounds__(256) k_kmap_bounds(const __grid_constant__ KmapBatch B) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ int64_t s_pre[KM_MAX_MAPS + 1];
    if (threadIdx.x == 0) {
        int64_t acc = 0;
        for (int m = 0; m < B.n_maps; ++m) {
            s_pre[m] = acc;
            const int64_t n_out = dev_count(B.d[m].n_out_cap, B.d[m].n_out_dev);
            acc += ((n_out + KM_BM - 1) / KM_BM) * 2 * B.d[m].kx * B.d[m].ky;
        }
        s_pre[B.n_maps] = acc;
    }
    __syncthreads();
    const int64_t total = s_pre[B.n_maps];
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
        int m = 0;
        while (s_pre[m + 1] <= v) ++m;
        const KmapDesc &p = B.d[m];
        const int G2 = 2 * p.kx * p.ky;
        const int64_t local = v - s_pre[m];
        const int64_t tile = local / G2;
        const int j = (int)(local - tile * G2), g = j >> 1, hi = j & 1;
        const int64_t n_out = dev_count(p.n_out_cap, p.n_out_dev);
        const int64_t n_in = dev_count(p.n_in_cap, p.n_in_dev);
        const int64_t row0 = tile * KM_BM;
        const int rows = (int)imin64(KM_BM, n_out - row0);
        const KeyT *in = static_cast<const KeyT *>(p.in), *out = static_cast<const KeyT *>(p.out);
        // packed(q) + packed(delta) in KeyT arithmetic: the planned headroom keeps the
        // true sum inside the key range, so the wrap-around addition is exact
        const KeyT q = hi ? (KeyT)(out[row0 + rows - 1] + (KeyT)group_delta(p, B.bits_y, B.bits_z, g, p.kz - 1) + (KeyT)1)
                          : (KeyT)(out[row0] + (KeyT)group_delta(p, B.bits_y, B.bits_z, g, 0));
        p.bounds[local] = (int32_t)lower_bound_g(in, n_in, q);
    }
}

// per-tile shared state of k_kmap_zdelta (the tile's OS / WS tables live in dynamic smem)
constexpr int KM_POOL = 4096;      // staged window keys per CTA (32 KB); a group that does not fit searches global
template <typename KeyT>
struct ZTile {
    KeyT q[KM_BM];                  // the tile's output keys
    uint32_t ordk[KM_BM];           // density-order direction bits per row
    int32_t cnt[SPC_MAX_KVOL];      // matches per weight offset
    int32_t wlo[25], wlen[25], woff[25];   // per offset group: window start / length / pool offset (-1: global)
    int64_t dq[SPC_MAX_KVOL];       // packed query delta of member mm of group g, at g * K + mm
    int32_t dsc[SPC_MAX_KVOL];      // its weight offset k | dense column + 1 << 8 | WS list + 1 << 16 | order bit + 1 << 24
    uint32_t mask[4];               // OS tile mask words
    int mslot[2];                   // map of this / the next tile (thread 0, parity-buffered)
};

__device__ __forceinline__ int tile_map(const int64_t *pre, int n_maps, int64_t v) {
    int m = 0;
    while (m + 1 < n_maps && pre[m + 1] <= v) ++m;
    return m;
}

// lower bound in a staged (shared) or global window; every call is counted in n_calls
// (the search-count law |V_q| K^2 of P:297 is checked against this counter)
template <typename KeyT, bool SM>
__device__ __forceinline__ int lb_win(const KeyT *a, int n, KeyT q, unsigned &n_calls) {
    ++n_calls;
    int lo = 0, len = n;
    while (len > 0) {
        const int half = len >> 1;
        KeyT v;
        if (SM) v = a[lo + half];
        else v = __ldg(a + lo + half);
        if (v < q) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return lo;
}

// one (offset group, 32-output chunk) task of a tile, one warp: the paper's z-delta search
// per output -- one lower_bound for the anchor query, then a forward cursor for the other
// K-1 members -- in the group's window of input keys.  Every stored entry is
// written to the tile's shared tables (-1 = no match): OS columns [row][K_dense], WS lists
// [list][row]; counts, mask bits and density-order bits go to shared accumulators.
// KT > 0: compile-time member count (unrolled: K = 1, 3, 5); KT = 0: runtime count k_rt
// (the even / non-cubic boxes of NEXT-3, kept out of line so the hot instantiations keep
// the kernel body small -- the build is instruction-issue bound)
template <typename KeyT, int KT, bool SM>
__device__ __forceinline__ int zdelta_chunk(ZTile<KeyT> &zt, int32_t *s_os, int32_t *s_ws, int KD, const KeyT *wk,
                                            int wl, int32_t lo, int g, int ch, int rows, int lane, unsigned &n_calls,
                                            int k_rt = KT) {
    const int K = KT > 0 ? KT : k_rt;
    const int lr = ch * 32 + lane;
    const bool valid = lr < rows;
    const KeyT q = valid ? zt.q[lr] : (KeyT)0;
    int pos = 0;
    if (valid) pos = lb_win<KeyT, SM>(wk, wl, (KeyT)(q + (KeyT)zt.dq[g * K]), n_calls);
    const int pos0 = pos;
    uint32_t key = 0;
#pragma unroll (KT > 0 ? KT : 1)
    for (int mm = 0; mm < K; ++mm) {   // members in ascending query order
        const KeyT query = (KeyT)(q + (KeyT)zt.dq[g * K + mm]);
        const int32_t dsc = zt.dsc[g * K + mm];
        bool match = false;
        if (valid) {
            KeyT v = 0;
            while (pos < wl && (v = (SM ? wk[pos] : __ldg(wk + pos))) < query) ++pos;
            match = pos < wl && v == query;
        }
        const int32_t j = match ? lo + pos : -1;
        const unsigned bal = __ballot_sync(0xffffffffu, match);
        const int col = ((dsc >> 8) & 0xff) - 1, l = ((dsc >> 16) & 0xff) - 1, ob = ((dsc >> 24) & 0x1f) - 1;
        if (valid) {
            if (col >= 0) s_os[lr * KD + col] = j;
            else if (l >= 0) s_ws[l * KM_BM + lr] = j;
        }
        if (lane == 0 && bal) {
            atomicAdd(&zt.cnt[dsc & 0xff], __popc(bal));
            if (col >= 0) atomicOr(&zt.mask[col >> 5], 1u << (col & 31));
        }
        if (match && ob >= 0) key |= 1u << ob;
    }
    if (key) atomicOr(&zt.ordk[lr], key);
    return pos - pos0;   // cursor advances (search-count statistics)
}

// (its own call counter: a reference into an out-of-line call would put the caller's
// counter in local memory on every path)
template <typename KeyT, bool SM>
__device__ __noinline__ int zdelta_chunk_rt(ZTile<KeyT> &zt, int32_t *s_os, int32_t *s_ws, int KD, const KeyT *wk,
                                            int wl, int32_t lo, int g, int ch, int rows, int lane, int K) {
    unsigned calls = 0;
    return zdelta_chunk<KeyT, 0, SM>(zt, s_os, s_ws, KD, wk, wl, lo, g, ch, rows, lane, calls, K);
}

// members per group (Kz) as a compile-time count
template <typename KeyT, bool SM>
__device__ __forceinline__ int zdelta_dispatch(int K, ZTile<KeyT> &zt, int32_t *s_os, int32_t *s_ws, int KD,
                                               const KeyT *wk, int wl, int32_t lo, int g, int ch, int rows, int lane,
                                               unsigned &n_calls) {
    if (K == 3) return zdelta_chunk<KeyT, 3, SM>(zt, s_os, s_ws, KD, wk, wl, lo, g, ch, rows, lane, n_calls);
    if (K == 5) return zdelta_chunk<KeyT, 5, SM>(zt, s_os, s_ws, KD, wk, wl, lo, g, ch, rows, lane, n_calls);
    if (K == 1) return zdelta_chunk<KeyT, 1, SM>(zt, s_os, s_ws, KD, wk, wl, lo, g, ch, rows, lane, n_calls);
    n_calls += ch * 32 + lane < rows ? 1u : 0u;   // the one anchor search per valid output
    return zdelta_chunk_rt<KeyT, SM>(zt, s_os, s_ws, KD, wk, wl, lo, g, ch, rows, lane, K);
}

constexpr int KM_MIN_BLOCKS = 4;
// one CTA per (map, tile of KM_BM outputs), grid-strided over every tile of every map of
// the batch.  Per tile: (1) every warp stages its share of the K^2 group windows
// [lo, hi) (k_kmap_bounds) into one shared pool, coalesced; (2) the warps share the
// (group, 32-output chunk) search tasks; (3) the tile leaves as contiguous streams: the OS
// block [rows x K_dense] (each entry written once, -1 for no match: no transpose pass,
// P:400) as 16-byte stores, each WS list's pairs compacted with one reservation per
// (tile, list) (warp ballots, no filter pass; halved for submanifold maps,
// P:418-421), the tile mask, per-offset counts and density-order keys.
template <typename KeyT>
__global__ void __launch_bounds__(KM_THREADS, KM_MIN_BLOCKS) k_kmap_zdelta(const __grid_constant__ KmapBatch B) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ int8_t s_dcol[KM_MAX_MAPS][SPC_MAX_KVOL];   // weight offset -> dense column / -1
    __shared__ int8_t s_lst[KM_MAX_MAPS][SPC_MAX_KVOL];    // weight offset -> WS list / -1
    __shared__ int64_t s_pre[KM_MAX_MAPS + 1];             // tile prefix over the maps
    __shared__ int64_t s_ordbase[KM_MAX_MAPS];
    __shared__ int64_t s_nout[KM_MAX_MAPS];
    __shared__ __align__(16) KeyT s_pool[KM_POOL];
    __shared__ ZTile<KeyT> zt;
    extern __shared__ __align__(16) int32_t s_tab[];        // [KM_BM x K_dense] OS, then [lists x KM_BM] WS

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // ---- prologue: per-map offset tables (planned on the host, make_plan) --------------
    for (int e = tid; e < B.n_maps * SPC_MAX_KVOL; e += KM_THREADS) {
        const int m = e / SPC_MAX_KVOL, k = e - m * SPC_MAX_KVOL;
        s_dcol[m][k] = B.d[m].dcol[k];
        s_lst[m][k] = B.d[m].lst[k];
    }
    if (tid == 0) {
        int64_t acc = 0, ob = 0;
        for (int m = 0; m < B.n_maps; ++m) {
            s_pre[m] = acc;
            const int64_t n_out = dev_count(B.d[m].n_out_cap, B.d[m].n_out_dev);
            s_nout[m] = n_out;
            acc += (n_out + KM_BM - 1) / KM_BM;
            s_ordbase[m] = ob;
            if (B.d[m].ord_idx >= 0) ob += n_out;
        }
        s_pre[B.n_maps] = acc;
        zt.mslot[0] = tile_map(s_pre, B.n_maps, blockIdx.x);
    }
    __syncthreads();
    const int64_t total = s_pre[B.n_maps];
    unsigned long long n_search = 0, n_probe = 0;
    unsigned n_calls = 0;   // lower_bound calls of this thread (lb_win)
    int stats_map = -1;
    // software pipeline: the next tile's output keys and window bounds are loaded into
    // registers while the current tile flushes (one global round trip off the tile chain)
    KeyT pf_q = 0;
    int32_t pf_lo = 0, pf_hi = 0;
    auto prefetch = [&](int64_t vn, int mn) {
        if (vn >= total) return;
        const KmapDesc &pn = B.d[mn];
        const int64_t tn = vn - s_pre[mn];
        const int rn = (int)imin64(KM_BM, s_nout[mn] - tn * KM_BM);
        if (tid < rn) pf_q = static_cast<const KeyT *>(pn.out)[tn * KM_BM + tid];
        const int Gn = pn.kx * pn.ky;
        if (lane < Gn) {
            const int2 b2 = *reinterpret_cast<const int2 *>(pn.bounds + (tn * Gn + lane) * 2);
            pf_lo = b2.x;
            pf_hi = b2.y;
        }
    };
    prefetch(blockIdx.x, zt.mslot[0]);

    uint32_t it = 0;
    for (int64_t v = blockIdx.x; v < total; v += gridDim.x, ++it) {
        const int m = zt.mslot[it & 1];
        if (tid == 0) zt.mslot[(it + 1) & 1] = tile_map(s_pre, B.n_maps, v + gridDim.x);
        const KmapDesc &p = B.d[m];
        const int8_t *dcol = s_dcol[m], *lstv = s_lst[m];
        const int64_t tile = v - s_pre[m];
        const int64_t row0 = tile * KM_BM;
        const int rows = (int)imin64(KM_BM, s_nout[m] - row0);
        const int K = p.kz, G = p.kx * p.ky, KD = p.k_dense;   // G groups of K members
        int32_t *s_os = s_tab;
        int32_t *s_ws = s_tab + KM_BM * KD;
        // ---- (1) tile state; group windows (every warp scans the <= 25 group sizes) ----
        if (tid < KM_BM) {
            zt.q[tid] = tid < rows ? pf_q : 0;
            zt.ordk[tid] = 0;
        }
        for (int e = tid; e < G * K; e += KM_THREADS) {
            zt.cnt[e] = 0;
            const int g = e / K, mm = e - g * K;
            const int k = g * K + (p.transposed ? K - 1 - mm : mm);   // weight offset (dz fastest)
            zt.dq[e] = group_delta(p, B.bits_y, B.bits_z, g, mm);
            const int col = dcol[k], l = lstv[k];
            const int ob = (p.ord_idx >= 0 && col >= 0) ? p.ord_cls[col] : -1;
            zt.dsc[e] = k | ((col + 1) << 8) | ((l + 1) << 16) | ((ob + 1) << 24);
        }
        if (tid < 4) zt.mask[tid] = 0;
        {
            int lo = 0, wl = 0;
            bool need = false;
            if (lane < G) {
                for (int mm = 0; mm < K; ++mm) {
                    const int k = lane * K + mm;
                    need |= dcol[k] >= 0 || lstv[k] >= 0;
                }
                if (need) {
                    lo = pf_lo;
                    wl = max(0, pf_hi - lo);
                }
            }
            int x = wl;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            const int off = x - wl;
            const bool fits = x <= B.pool_keys;
            if (warp == 0 && lane < G) {
                zt.wlo[lane] = lo;
                zt.wlen[lane] = need ? wl : -1;   // -1: group not needed
                zt.woff[lane] = fits ? off : -1;
            }
            // stage: warp w copies groups w, w + 8, ...
            for (int gg = warp; gg < G; gg += KM_WARPS) {
                const int glo = __shfl_sync(0xffffffffu, lo, gg), gwl = __shfl_sync(0xffffffffu, wl, gg);
                const int goff = __shfl_sync(0xffffffffu, off, gg);
                if (!__shfl_sync(0xffffffffu, fits ? 1 : 0, gg)) continue;
                const KeyT *src = static_cast<const KeyT *>(p.in) + glo;
                KeyT *dst = s_pool + goff;
                int e = lane;
                for (; e + 96 < gwl; e += 128) {
                    const KeyT a0 = __ldg(src + e), a1 = __ldg(src + e + 32), a2 = __ldg(src + e + 64),
                               a3 = __ldg(src + e + 96);
                    dst[e] = a0; dst[e + 32] = a1; dst[e + 64] = a2; dst[e + 96] = a3;
                }
                for (; e < gwl; e += 32) dst[e] = __ldg(src + e);
            }
        }
        __syncthreads();
        if (p.stats && stats_map != m) {   // flush the stats of the previous map
            n_search += n_calls;
            n_calls = 0;
            for (int o = 16; o > 0; o >>= 1) {
                n_search += __shfl_xor_sync(0xffffffffu, n_search, o);
                n_probe += __shfl_xor_sync(0xffffffffu, n_probe, o);
            }
            if (stats_map >= 0 && lane == 0) {
                atomicAdd(&B.d[stats_map].stats[0], n_search);
                atomicAdd(&B.d[stats_map].stats[1], n_probe);
            }
            n_search = n_probe = 0;
            stats_map = m;
        }
        // ---- (2) search tasks: (group, chunk) -------------------------------------------
        const int nch = (rows + 31) / 32;
        for (int t = warp; t < G * nch; t += KM_WARPS) {
            const int g = t / nch, ch = t - g * nch;
            const int wl = zt.wlen[g];
            if (wl < 0) continue;
            const int32_t lo = zt.wlo[g];
            const int off = zt.woff[g];
            int adv;
            if (off >= 0) {
                const KeyT *wk = s_pool + off;
                adv = zdelta_dispatch<KeyT, true>(K, zt, s_os, s_ws, KD, wk, wl, lo, g, ch, rows, lane, n_calls);
            } else {
                const KeyT *wk = static_cast<const KeyT *>(p.in) + lo;
                adv = zdelta_dispatch<KeyT, false>(K, zt, s_os, s_ws, KD, wk, wl, lo, g, ch, rows, lane, n_calls);
            }
            n_probe += (unsigned long long)adv;
        }
        __syncthreads();
        prefetch(v + gridDim.x, zt.mslot[(it + 1) & 1]);
        // ---- (3) flush ------------------------------------------------------------------
        if (KD > 0) {   // OS block: rows x K_dense contiguous int32 (16-byte aligned: 512 * tile * KD)
            const int n_el = rows * KD;
            int32_t *dst = p.os + row0 * KD;
            const int n4 = n_el >> 2;
            for (int e = tid; e < n4; e += KM_THREADS)
                __stcs(reinterpret_cast<int4 *>(dst) + e, reinterpret_cast<const int4 *>(s_os)[e]);
            for (int e = 4 * n4 + tid; e < n_el; e += KM_THREADS) __stcs(dst + e, s_os[e]);
            if (tid < p.tile_words) p.tile_mask[tile * p.tile_words + tid] = zt.mask[tid];
        }
        {   // WS lists: warp w compacts lists w, w + 8, ... (one reservation per tile and list)
            int nl = 0;
            for (int k = 0; k < G * K; ++k) nl = max(nl, lstv[k] + 1);
            for (int l = warp; l < nl; l += KM_WARPS) {
                const int32_t *col = s_ws + l * KM_BM;
                int32_t jv[KM_BM / 32];
                unsigned bal[KM_BM / 32];
                int c = 0;
#pragma unroll
                for (int ch = 0; ch < KM_BM / 32; ++ch) {
                    const int lr = ch * 32 + lane;
                    jv[ch] = lr < rows ? col[lr] : -1;
                    bal[ch] = __ballot_sync(0xffffffffu, jv[ch] >= 0);
                    c += __popc(bal[ch]);
                }
                if (c == 0) continue;
                int b = 0;
                if (lane == 0) b = atomicAdd(&p.counts[SPC_MAX_KVOL + l], c);
                b = __shfl_sync(0xffffffffu, b, 0);
                int2 *dst = p.pairs + (int64_t)l * p.list_stride;
#pragma unroll
                for (int ch = 0; ch < KM_BM / 32; ++ch) {
                    if (jv[ch] >= 0)
                        __stcs(dst + b + __popc(bal[ch] & lanemask_lt()), make_int2(jv[ch], (int32_t)(row0 + ch * 32 + lane)));
                    b += __popc(bal[ch]);
                }
            }
        }
        for (int k = tid; k < G * K; k += KM_THREADS)
            if (zt.cnt[k]) atomicAdd(&p.counts[k], zt.cnt[k]);
        if (p.ord_idx >= 0 && tid < rows)
            __stcs(reinterpret_cast<unsigned long long *>(B.ord_keys) + s_ordbase[m] + row0 + tid,
                   (unsigned long long)(((uint64_t)p.ord_idx << B.ord_key_bits) | zt.ordk[tid]));
        __syncthreads();
    }
    if (stats_map >= 0) {
        n_search += n_calls;
        for (int o = 16; o > 0; o >>= 1) {
            n_search += __shfl_xor_sync(0xffffffffu, n_search, o);
            n_probe += __shfl_xor_sync(0xffffffffu, n_probe, o);
        }
        if (lane == 0) {
            atomicAdd(&B.d[stats_map].stats[0], n_search);
            atomicAdd(&B.d[stats_map].stats[1], n_probe);
        }
    }
}

// ------------------------------------------------------------------------------------
// ablation (SPC_KMAP_SIMPLE_BSEARCH): the paper's "Simple BSearch" mapping baseline
// (P:257-259): one independent binary search over the whole sorted input per (output,
// offset), |V_q| K^3 searches.  One thread per (offset k, output i), i fastest, so a warp
// holds 32 consecutive outputs of one offset (one ballot for the counts and tile mask).
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_kmap_bsearch(const __grid_constant__ KmapDesc p, int bits_y, int bits_z) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    const int64_t n_out = dev_count(p.n_out_cap, p.n_out_dev);
    const int64_t n_in = dev_count(p.n_in_cap, p.n_in_dev);
    const int64_t n_pad = (n_out + 31) & ~int64_t(31);
    const int kv = p.kx * p.ky * p.kz;
    const int lane = threadIdx.x & 31;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < kv * n_pad; e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e / n_pad);
        const int64_t i = e - k * n_pad;
        const int col = p.dcol[k];
        const int ex = k / (p.ky * p.kz) + p.lox, ey = (k / p.kz) % p.ky + p.loy, ez = k % p.kz + p.loz;
        int64_t d = (int64_t)ex * p.spacing * (1ll << (bits_y + bits_z)) + (int64_t)ey * p.spacing * (1ll << bits_z) +
                    (int64_t)ez * p.spacing;
        if (p.transposed) d = -d;
        const bool valid = i < n_out;
        bool match = false;
        int32_t j = -1;
        if (valid) {
            const uint64_t *in = static_cast<const uint64_t *>(p.in);
            const uint64_t q = static_cast<const uint64_t *>(p.out)[i] + (uint64_t)d;
            const int64_t pos = lower_bound_g(in, n_in, q);
            match = pos < n_in && __ldg(in + pos) == q;
            if (match) j = (int32_t)pos;
            p.os[i * p.k_dense + col] = j;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, match), vb = __ballot_sync(0xffffffffu, valid);
        if (lane == 0) {
            if (bal) {
                atomicAdd(&p.counts[k], __popc(bal));
                atomicOr(&p.tile_mask[(i / KM_BM) * p.tile_words + (col >> 5)], 1u << (col & 31));
            }
            if (p.stats && vb) atomicAdd(&p.stats[0], (unsigned long long)__popc(vb));
        }
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
constexpr int ORD_MAX = 16;   // ordered maps per network build (tag bits: ceil(log2 n))
struct OrderJob {
    const int32_t *os;
    int32_t *os_ord;
    uint32_t *mask_ord;
    int32_t *rows;
    int32_t *tile_order;      // [2][tiles128]
    const int64_t *n_dev;
    int64_t n_cap;
    int64_t tile0;            // first permute CTA of this map
    int k_dense, words;
};
struct OrderBatch {
    int n_jobs;
    OrderJob j[ORD_MAX];
};

// the grouped order's scratch: key array (written by the z-delta build), live total,
// sorted keys / positions, radix workspace
struct OrderScratch {
    int64_t *total;
    uint64_t *keys, *keys_sorted;
    int32_t *pos;
    void *rws;
    size_t rws_bytes;
    bool ok;
};
static OrderScratch order_scratch(void *base, size_t bytes, int64_t rows_cap) {
    OrderScratch o{};
    Bump b(base, bytes);
    o.total = b.take<int64_t>(4);
    o.keys = b.take<uint64_t>((size_t)rows_cap);
    o.keys_sorted = b.take<uint64_t>((size_t)rows_cap);
    o.pos = b.take<int32_t>((size_t)rows_cap);
    o.rws_bytes = radix_sort_workspace(rows_cap, true);
    o.rws = b.take<uint8_t>(o.rws_bytes);
    o.ok = b.ok();
    return o;
}
static int ord_tag_bits(int n_jobs) {
    int t = 0;
    while ((1 << t) < n_jobs) ++t;
    return t;
}
// key = [map tag | 16 - popcount(dirs) (5 bits) | dirs (16 bits)]: heaviest rows first, then
// grouped by direction pattern; <= 24 bits = 3 radix passes
constexpr int ORD_DIR_BITS = 16, ORD_TAG_SHIFT = 21;
static int ord_key_bits(int n_jobs) { (void)n_jobs; return ORD_TAG_SHIFT; }

// weight field of every key (the build ORs only the direction bits in)
__global__ void k_ord_weight(uint64_t *__restrict__ keys, const int64_t *total) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    const int64_t n = *total;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        const uint32_t dirs = (uint32_t)k & ((1u << ORD_DIR_BITS) - 1);
        keys[i] = k | ((uint64_t)(ORD_DIR_BITS - __popc(dirs)) << ORD_DIR_BITS);
    }
}

__device__ __forceinline__ int64_t ord_base(const OrderBatch &B, int job, int64_t &n_job) {
    int64_t base = 0;
    for (int q = 0; q < job; ++q) base += dev_count(B.j[q].n_cap, B.j[q].n_dev);
    n_job = dev_count(B.j[job].n_cap, B.j[job].n_dev);
    return base;
}

// one CTA per 128-row tile of one map: row p of the ordered table = row rows[p] of the
// canonical one.  Each warp copies its 32 rows as one flat range of 32*k_dense elements
// (independent loads, coalesced stores); tile mask words from per-lane column masks.
__global__ void __launch_bounds__(128) k_ord_permute(const __grid_constant__ OrderBatch B,
                                                     const int32_t *__restrict__ sorted_pos) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
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
    const int KD = J.k_dense;
    const int nrows = (int)imin64(32, n - (p0 + w * 32));
    uint32_t m[4] = {0u, 0u, 0u, 0u};
    if (nrows > 0) {
        const int total = nrows * KD;
        int32_t *dst = J.os_ord + (p0 + w * 32) * KD;
#pragma unroll 4
        for (int e = lane; e < total; e += 32) {
            const int r = e / KD, c = e - r * KD;
            const int32_t v = J.os[(int64_t)src_s[w * 32 + r] * KD + c];
            dst[e] = v;
            if (v >= 0) m[c >> 5] |= 1u << (c & 31);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t r = __reduce_or_sync(0xffffffffu, m[q]);
        if (lane == 0) wm[w][q] = r;
    }
    __syncthreads();
    if (threadIdx.x < J.words) {
        const int q = threadIdx.x;
        J.mask_ord[(p0 / 128) * J.words + q] = wm[0][q] | wm[1][q] | wm[2][q] | wm[3][q];
    }
}

// tile orders of one map (CTA pair per map: 128-row tiles, 256-row tiles): tiles by
// descending weight = popcount of the tile mask (the number of offset slices a conv CTA
// runs for it), so a dynamic scheduler claiming them in this order balances like LPT.
// Equal weights in any order (the conv's result does not depend on the tile order).
__global__ void __launch_bounds__(1024) k_ord_tiles(const __grid_constant__ OrderBatch B) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ int hist[SPC_MAX_KVOL + 2];
    const OrderJob &J = B.j[blockIdx.x >> 1];
    const int T = (blockIdx.x & 1) ? 256 : 128, f = T / 128;
    const int64_t n = dev_count(J.n_cap, J.n_dev);
    const int64_t tiles128 = (J.n_cap + 127) / 128;
    const int64_t nt = (n + T - 1) / T, nt128 = (n + 127) / 128;
    int32_t *order = J.tile_order + (f == 2 ? tiles128 : 0);
    int32_t *wout = J.tile_order + 2 * tiles128 + (f == 2 ? tiles128 : 0);   // weights in claim order
    for (int i = threadIdx.x; i < SPC_MAX_KVOL + 2; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    auto weight = [&](int64_t t) {
        int w = 0;
        for (int q = 0; q < J.words; ++q) {
            uint32_t m = 0;
            for (int h = 0; h < f; ++h)
                if (t * f + h < nt128) m |= J.mask_ord[(t * f + h) * J.words + q];
            w += __popc(m);
        }
        return min(w, SPC_MAX_KVOL);
    };
    for (int64_t t = threadIdx.x; t < nt; t += blockDim.x) atomicAdd(&hist[SPC_MAX_KVOL - weight(t)], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int i = 0; i <= SPC_MAX_KVOL; ++i) {
            const int c = hist[i];
            hist[i] = acc;
            acc += c;
        }
    }
    __syncthreads();
    for (int64_t t = threadIdx.x; t < nt; t += blockDim.x) {
        const int w = weight(t);
        const int at = atomicAdd(&hist[SPC_MAX_KVOL - w], 1);
        order[at] = (int32_t)t;
        wout[at] = w;
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

// sort the keys of `jobs` (already written by the z-delta build) and permute their OS tables
static spc_status run_orders(const std::vector<OrderJob> &jobs, const OrderScratch &o, int64_t rows_cap,
                             cudaStream_t st) {
    if (jobs.empty() || rows_cap == 0) return SPC_OK;
    if (!o.ok) return fail(SPC_ERR_WORKSPACE, "kernel-map density order: scratch too small");
    OrderBatch B;
    memset(&B, 0, sizeof(B));
    B.n_jobs = (int)jobs.size();
    int64_t tiles = 0;
    for (int q = 0; q < B.n_jobs; ++q) {
        B.j[q] = jobs[q];
        B.j[q].tile0 = tiles;
        tiles += (B.j[q].n_cap + 127) / 128;
    }
    SPC_CUDA(launch_pdl(k_ord_weight, dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((rows_cap + 255) / 256, 4 * (int64_t)num_sms()))), dim3(256), 0, st, o.keys, o.total));
    SPC_LAUNCH_CHECK("k_ord_weight");
    spc_status s = radix_sort(o.keys, nullptr, rows_cap, o.total, ORD_TAG_SHIFT + ord_tag_bits(B.n_jobs), o.keys_sorted,
                              o.pos, o.rws, o.rws_bytes, st, false);
    if (s != SPC_OK) return s;
    SPC_CUDA(launch_pdl(k_ord_permute, dim3((unsigned)tiles), dim3(128), 0, st, B, o.pos));
    SPC_LAUNCH_CHECK("k_ord_permute");
    SPC_CUDA(launch_pdl(k_ord_tiles, dim3((unsigned)(2 * B.n_jobs)), dim3(1024), 0, st, B));
    SPC_LAUNCH_CHECK("k_ord_tiles");
    return SPC_OK;
}

// ------------------------------------------------------------------------------------
// host: plan (offset tables, dense/sparse split, lists) and entry points
// ------------------------------------------------------------------------------------
struct KmapPlan {
    int kk[3] = {0, 0, 0}, lo[3] = {0, 0, 0};   // offset box: sizes and first offset per axis (units)
    int reach_units = 0;                        // max |e| over the box (the map's reach / spacing)
    bool symmetric = false;                     // every size odd: centred box, k <-> k_vol-1-k mirrors
    int k_vol = 0, k_dense = 0, n_lists = 0, halved = 0, t_eff = 0, spacing = 1, centre_col = -1;
    int16_t dense_k[SPC_MAX_KVOL], list_k[SPC_MAX_KVOL];
    int8_t list_mirror[SPC_MAX_KVOL];
    int16_t dense_col[SPC_MAX_KVOL], list_id[SPC_MAX_KVOL];
    int8_t ord_cls[SPC_MAX_KVOL];   // density-order key bit of each dense column (-1: none)
    uint8_t group_needed[25];
};

static spc_status make_plan(const spc_geom &g, int32_t t, uint32_t flags, KmapPlan &pl) {
    // offset box: Delta(K, s_p) for odd cubic K; per-axis sizes and even sizes
    // ({0 .. K-1}, reading E1) are the generalisation of SURVEY NEXT-3
    const int ks[3] = {g.kernel_size, g.kernel_size_y > 0 ? g.kernel_size_y : g.kernel_size,
                       g.kernel_size_z > 0 ? g.kernel_size_z : g.kernel_size};
    for (int a = 0; a < 3; ++a)
        if (ks[a] < 1 || ks[a] > 5)
            return fail(SPC_ERR_UNSUPPORTED, "kernel sizes must be in 1..5, got " + std::to_string(ks[a]));
    if (g.stride < 1 || g.dilation < 1 || g.tensor_stride < 1)
        return fail(SPC_ERR_INVALID_ARG, "stride, dilation and tensor_stride must be >= 1");
    if (g.transposed && g.stride == 1)
        return fail(SPC_ERR_INVALID_ARG, "a transposed map needs stride > 1");
    pl.symmetric = true;
    pl.reach_units = 0;
    for (int a = 0; a < 3; ++a) {
        pl.kk[a] = ks[a];
        pl.lo[a] = ks[a] % 2 ? -(ks[a] - 1) / 2 : 0;
        pl.symmetric &= ks[a] % 2 == 1;
        pl.reach_units = std::max(pl.reach_units, std::max(-pl.lo[a], pl.lo[a] + ks[a] - 1));
    }
    pl.k_vol = ks[0] * ks[1] * ks[2];
    pl.spacing = g.tensor_stride * g.dilation;
    int l1max = 0;
    for (int a = 0; a < 3; ++a) l1max += std::max(-pl.lo[a], pl.lo[a] + ks[a] - 1);
    pl.t_eff = (t < 0 || t > l1max + 1) ? l1max + 1 : t;
    const bool subm = g.stride == 1 && !g.transposed;
    // halving needs the mirror pairs k <-> k_vol-1-k of a centred box
    pl.halved = (flags & SPC_KMAP_HALVE_SYMMETRIC) && subm && pl.symmetric ? 1 : 0;
    const int centre = pl.symmetric ? (pl.k_vol - 1) / 2 : -1;   // the zero offset, if the box has it
    pl.k_dense = pl.n_lists = 0;
    pl.centre_col = -1;
    for (int k = 0; k < pl.k_vol; ++k) {
        int ex = k / (ks[1] * ks[2]) + pl.lo[0], ey = (k / ks[2]) % ks[1] + pl.lo[1], ez = k % ks[2] + pl.lo[2];
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
            const int k = pl.dense_k[c];
            const int r = rank[k];
            if (r < 0 || ncls <= 16) {
                pl.ord_cls[c] = (int8_t)r;   // every direction pair its own bit (K = 3: 13)
                continue;
            }
            // more pairs than bits (K = 5: 62): fold by geometry, not by index -- the axes
            // the offset moves along (7 patterns) x inner / outer ring (|e|_inf 1 or 2): rows
            // of one surface orientation share bits (r % 16 merged unrelated directions)
            const int ex = k / (ks[1] * ks[2]) + pl.lo[0], ey = (k / ks[2]) % ks[1] + pl.lo[1], ez = k % ks[2] + pl.lo[2];
            const int mask = (ex != 0) << 2 | (ey != 0) << 1 | (ez != 0);
            const int linf = std::max(std::abs(ex), std::max(std::abs(ey), std::abs(ez)));
            pl.ord_cls[c] = (int8_t)(mask == 0 ? -1 : (mask - 1) + 7 * (linf >= 2 ? 1 : 0));
        }
    }
    for (int gi = 0; gi < ks[0] * ks[1]; ++gi) {
        bool need = false;
        for (int m = 0; m < ks[2]; ++m) {
            int k = gi * ks[2] + m;
            need |= pl.dense_col[k] >= 0 || pl.list_id[k] >= 0;
        }
        pl.group_needed[gi] = need;
    }
    return SPC_OK;
}

struct KmapLayout {
    size_t os, pairs, counts, mask, stats, bounds, total;
    size_t rows, os_ord, mask_ord, tile_order, scratch, scratch_bytes;   // density order
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
    L.bounds = take(sizeof(int32_t) * (size_t)L.tiles * 2 * pl.kk[0] * pl.kk[1]);
    if (wants_order(pl, flags)) {
        L.rows = take(sizeof(int32_t) * (size_t)n_out);
        L.os_ord = take(sizeof(int32_t) * (size_t)n_out * pl.k_dense);
        L.mask_ord = take(sizeof(uint32_t) * (size_t)(L.tiles * L.words));
        L.tile_order = take(sizeof(int32_t) * 4 * (size_t)L.tiles);   // orders + weights
        if (scratch) {
            L.scratch_bytes = order_scratch_bytes(n_out);
            L.scratch = take(L.scratch_bytes);
        }
    }
    L.total = align_up(off, 256);
    return L;
}



struct DeferState {
    bool active = false;
    KmapBatch b;
    int max_kd = 0;
    int64_t tiles = 0;
    std::vector<OrderJob> orders;
    OrderScratch scratch{};    // density-order scratch of the batch
    int64_t order_rows = 0;    // its row capacity
    bool flushed = false;      // a full batch was launched early (later maps: no density order)
    bool batch_orders = false; // the current batch holds ordered maps (it owns the order scratch)
};
static thread_local DeferState g_defer;
static spc_status launch_kmaps(const KmapBatch &b, int max_kd, int64_t tiles, cudaStream_t st);

// a full batch (KM_MAX_MAPS maps, one grid-constant descriptor table) is launched as soon
// as the next map arrives; the density-order key width is fixed by then, so maps added
// after an early launch are built without a density order (they stay valid maps)
static spc_status defer_flush(cudaStream_t st) {
    KmapBatch &b = g_defer.b;
    if (g_defer.batch_orders) {
        if (!g_defer.scratch.ok) return fail(SPC_ERR_WORKSPACE, "network kmaps: density-order scratch too small");
        b.ord_keys = g_defer.scratch.keys;
        b.ord_total = g_defer.scratch.total;
        b.ord_key_bits = ord_key_bits((int)g_defer.orders.size());
    }
    spc_status s = launch_kmaps(b, g_defer.max_kd, g_defer.tiles, st);
    memset(&g_defer.b, 0, sizeof(g_defer.b));
    g_defer.batch_orders = false;
    g_defer.max_kd = 0;
    g_defer.tiles = 0;
    g_defer.flushed = true;
    return s;
}

static void fill_desc(KmapDesc &d, const spc_kmap &km, const KmapPlan &pl, int32_t *bounds) {
    memset(&d, 0, sizeof(d));
    d.bounds = bounds;
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
    d.kx = (int32_t)pl.kk[0];
    d.ky = (int32_t)pl.kk[1];
    d.kz = (int32_t)pl.kk[2];
    d.lox = (int32_t)pl.lo[0];
    d.loy = (int32_t)pl.lo[1];
    d.loz = (int32_t)pl.lo[2];
    d.k_dense = pl.k_dense;
    d.tile_words = km.tile_words;
    d.t_eff = pl.t_eff;
    d.transposed = km.geom.transposed;
    d.halved = pl.halved;
    d.ord_idx = -1;
    for (int c = 0; c < pl.k_dense; ++c) d.ord_cls[c] = pl.ord_cls[c];
    for (int k = 0; k < SPC_MAX_KVOL; ++k) {
        d.dcol[k] = (int8_t)(k < pl.k_vol ? pl.dense_col[k] : -1);
        d.lst[k] = (int8_t)(k < pl.k_vol ? pl.list_id[k] : -1);
    }
}

static spc_status launch_kmaps(const KmapBatch &b0, int max_k_dense, int64_t max_tiles, cudaStream_t st) {
    KmapBatch b = b0;
    b.pool_keys = (int)std::max<int64_t>(0, std::min<int64_t>(KM_POOL, option(SPC_OPT_KMAP_POOL_KEYS)));
    SPC_CUDA(launch_pdl(k_kmap_prep, dim3(b.n_maps > 0 ? b.n_maps : 1), dim3(256), 0, st, b));
    SPC_LAUNCH_CHECK("k_kmap_prep");
    {
        int64_t items = 0;
        for (int m = 0; m < b.n_maps; ++m) items += ((b.d[m].n_out_cap + KM_BM - 1) / KM_BM) * 2 * b.d[m].kx * b.d[m].ky;
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, 16 * (int64_t)num_sms()));
        if (b.key_bytes == 4) SPC_CUDA(launch_pdl(k_kmap_bounds<uint32_t>, dim3(g), dim3(256), 0, st, b));
        else SPC_CUDA(launch_pdl(k_kmap_bounds<uint64_t>, dim3(g), dim3(256), 0, st, b));
        SPC_LAUNCH_CHECK("k_kmap_bounds");
    }
    // one CTA per (map, tile); the OS block of a tile is staged in dynamic shared memory
    int max_cols = 1;
    for (int m = 0; m < b.n_maps; ++m) {
        int nl = 0;
        for (int k = 0; k < SPC_MAX_KVOL; ++k) nl = std::max(nl, (int)b.d[m].lst[k] + 1);
        max_cols = std::max(max_cols, (int)b.d[m].k_dense + nl);
    }
    (void)max_k_dense;
    const size_t dsm = (size_t)KM_BM * max_cols * sizeof(int32_t);
    void (*kz)(KmapBatch) = b.key_bytes == 4 ? k_kmap_zdelta<uint32_t> : k_kmap_zdelta<uint64_t>;
    static size_t dsm_set[2][64] = {};   // per key width and device
    const int dev = current_device();
    if (dsm > dsm_set[b.key_bytes == 4][dev]) {
        SPC_CUDA(cudaFuncSetAttribute(kz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
        dsm_set[b.key_bytes == 4][dev] = dsm;
    }
    int per_sm = 0;
    SPC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kz, KM_THREADS, dsm));
    int64_t tiles = 0;
    for (int m = 0; m < b.n_maps; ++m) tiles += (b.d[m].n_out_cap + KM_BM - 1) / KM_BM;
    (void)max_tiles;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms() * std::max(1, per_sm)));
    SPC_CUDA(launch_pdl(kz, dim3((unsigned)grid), dim3(KM_THREADS), dsm, st, b));
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
// one build for 64-bit (key_bytes 8) or 32-bit single-scan (key_bytes 4) sorted keys
static spc_status build_kmap(const void *in_keys, int64_t n_in, const int64_t *n_in_dev, const void *out_keys,
                             int64_t n_out, const int64_t *n_out_dev, spc_pack_spec spec, spc_geom geom, int32_t t,
                             uint32_t flags, void *buf, size_t buf_bytes, uint32_t *status, spc_kmap *kmap_out,
                             void *stream, int key_bytes) {
    SPC_CHECK_ARG(kmap_out, "null kmap_out");
    SPC_CHECK_ARG(n_in >= 0 && n_out >= 0, "negative size");
    SPC_CHECK_ARG(n_in < INT32_MAX && n_out < INT32_MAX, "sizes must fit int32 indices");
    SPC_CHECK_ARG((in_keys || n_in == 0) && (out_keys || n_out == 0), "null keys");
    // symmetric halving needs ONE coordinate set: the same key array as input
    // and output (a range shard of a submanifold layer has different in / out index spaces)
    if ((flags & SPC_KMAP_HALVE_SYMMETRIC) && geom.stride == 1 && !geom.transposed &&
        (in_keys != out_keys || n_in != n_out || n_in_dev != n_out_dev))
        return fail(SPC_ERR_INVALID_ARG, "spc_build_kmap: SPC_KMAP_HALVE_SYMMETRIC needs in_keys == out_keys");
    KmapPlan pl;
    spc_status s = make_plan(geom, t, flags, pl);
    if (s != SPC_OK) return s;
    const KmapLayout L = layout_of(pl, n_out, flags, !g_defer.active);
    SPC_CHECK_ARG(buf && ((uintptr_t)buf % 256) == 0, "buf must be non-null and 256-byte aligned");
    if (buf_bytes < L.total) return fail(SPC_ERR_WORKSPACE, "spc_build_kmap: buffer too small");
    // reach check (reading A4): spc_pack_sort guarantees every key leaves `spec.reach`
    // (and out_stride - 1 below) of headroom in each field; a map reaching further could
    // carry or borrow into a neighbouring field, so it is refused, never truncated
    const int64_t reach = (int64_t)pl.reach_units * pl.spacing;
    if (reach > spec.reach)
        return fail(SPC_ERR_RANGE, "spc_build_kmap: kernel reach r*tensor_stride*dilation = " + std::to_string(reach) +
                                       " exceeds the planned spec.reach = " + std::to_string(spec.reach));
    if ((int64_t)geom.tensor_stride * geom.stride > spec.out_stride)
        return fail(SPC_ERR_RANGE, "spc_build_kmap: coarse stride " +
                                       std::to_string((int64_t)geom.tensor_stride * geom.stride) +
                                       " exceeds the planned spec.out_stride = " + std::to_string(spec.out_stride));
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
    km.in_keys = static_cast<const uint64_t *>(in_keys);     // (uint32 keys when key_bits == 32)
    km.out_keys = static_cast<const uint64_t *>(out_keys);
    km.key_bits = 8 * key_bytes;
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
    // a batch orders at most ORD_MAX maps (one tag each); later ones keep the canonical order
    if (g_defer.active && g_defer.b.n_maps >= KM_MAX_MAPS) {
        spc_status fs = defer_flush(st);
        if (fs != SPC_OK) return fs;
    }
    const bool order = wants_order(pl, flags) && n_out > 0 &&
                       (!g_defer.active || (g_defer.orders.size() < ORD_MAX && !g_defer.flushed));
    if (order) {
        km.os_rows = reinterpret_cast<int32_t *>(base + L.rows);
        km.os_table_ord = reinterpret_cast<int32_t *>(base + L.os_ord);
        km.tile_mask_ord = reinterpret_cast<uint32_t *>(base + L.mask_ord);
        km.tile_order = reinterpret_cast<int32_t *>(base + L.tile_order);
        job.tile_order = km.tile_order;
        job.os = km.os_table;
        job.os_ord = km.os_table_ord;
        job.mask_ord = km.tile_mask_ord;
        job.rows = km.os_rows;
        job.n_dev = n_out_dev;
        job.n_cap = n_out;
        job.k_dense = pl.k_dense;
        job.words = L.words;
    }
    if (n_out == 0) {
        SPC_CUDA(cudaMemsetAsync(base + L.counts, 0, L.stats + 2 * sizeof(unsigned long long) - L.counts, st));
        return SPC_OK;
    }
    if ((flags & SPC_KMAP_CHECK_SORTED) && status) {
        s = flag_unsorted(in_keys, key_bytes, n_in, n_in_dev, status, st);
        if (s == SPC_OK) s = flag_unsorted(out_keys, key_bytes, n_out, n_out_dev, status, st);
        if (s != SPC_OK) return s;
    }

    if (g_defer.active) {
        // network-wide phase 2: collect, launch once in kmap_defer_end()
        if (key_bytes != 8) return fail(SPC_ERR_UNSUPPORTED, "network-wide kernel maps use 64-bit keys");
        KmapBatch &b = g_defer.b;
        if (b.n_maps == 0) {
            b.key_bytes = 8;
            b.bits_y = spec.bits_y;
            b.bits_z = spec.bits_z;
            b.work_ctr = reinterpret_cast<unsigned int *>(base + L.stats) + 4;
        } else if (b.bits_y != spec.bits_y || b.bits_z != spec.bits_z) {
            return fail(SPC_ERR_INVALID_ARG, "batched kernel maps must share one pack spec");
        }
        KmapDesc &d = b.d[b.n_maps++];
        fill_desc(d, km, pl, reinterpret_cast<int32_t *>(base + L.bounds));
        g_defer.max_kd = std::max(g_defer.max_kd, pl.k_dense);
        g_defer.tiles += (int64_t)L.tiles;
        if (order) {
            d.ord_idx = (int32_t)g_defer.orders.size();
            g_defer.orders.push_back(job);
            g_defer.batch_orders = true;
        }
        return SPC_OK;
    }
    if (flags & SPC_KMAP_SIMPLE_BSEARCH) {
        // ablation baseline: all-OS maps only, no density order
        if (key_bytes != 8) return fail(SPC_ERR_UNSUPPORTED, "SPC_KMAP_SIMPLE_BSEARCH uses 64-bit keys");
        if (pl.n_lists != 0) return fail(SPC_ERR_UNSUPPORTED, "SPC_KMAP_SIMPLE_BSEARCH needs an all-OS t (SPC_T_ALL_OS)");
        KmapDesc d;
        fill_desc(d, km, pl, reinterpret_cast<int32_t *>(base + L.bounds));
        km.os_rows = nullptr;
        km.os_table_ord = nullptr;
        km.tile_mask_ord = nullptr;
        km.tile_order = nullptr;
        SPC_CUDA(cudaMemsetAsync(base + L.counts, 0, L.stats + 2 * sizeof(unsigned long long) - L.counts, st));
        const int64_t items = (int64_t)pl.k_vol * ((n_out + 31) & ~int64_t(31));
        SPC_CUDA(launch_pdl(k_kmap_bsearch, dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, 32 * (int64_t)num_sms()))), dim3(256), 0, st, d, spec.bits_y, spec.bits_z));
        SPC_LAUNCH_CHECK("k_kmap_bsearch");
        return SPC_OK;
    }
    KmapBatch b;
    memset(&b, 0, sizeof(b));
    b.n_maps = 1;
    b.bits_y = spec.bits_y;
    b.bits_z = spec.bits_z;
    b.work_ctr = reinterpret_cast<unsigned int *>(base + L.stats) + 4;   // scratch after the stats
    b.key_bytes = key_bytes;
    fill_desc(b.d[0], km, pl, reinterpret_cast<int32_t *>(base + L.bounds));
    OrderScratch os{};
    if (order) {
        os = order_scratch(base + L.scratch, L.scratch_bytes, n_out);
        if (!os.ok) return fail(SPC_ERR_WORKSPACE, "spc_build_kmap: density-order scratch too small");
        b.d[0].ord_idx = 0;
        b.ord_keys = os.keys;
        b.ord_total = os.total;
        b.ord_key_bits = ord_key_bits(1);
    }
    s = launch_kmaps(b, pl.k_dense, (int64_t)L.tiles, st);
    if (s == SPC_OK && order) s = run_orders(std::vector<OrderJob>{job}, os, n_out, st);
    return s;
}
}  // namespace spc

extern "C" spc_status spc_build_kmap(const uint64_t *in_keys, int64_t n_in, const int64_t *n_in_dev,
                                     const uint64_t *out_keys, int64_t n_out, const int64_t *n_out_dev,
                                     spc_pack_spec spec, spc_geom geom, int32_t t, uint32_t flags, void *buf,
                                     size_t buf_bytes, uint32_t *status, spc_kmap *kmap_out, void *stream) {
    return build_kmap(in_keys, n_in, n_in_dev, out_keys, n_out, n_out_dev, spec, geom, t, flags, buf, buf_bytes, status,
                      kmap_out, stream, 8);
}

extern "C" spc_status spc_build_kmap32(const uint32_t *in_keys, int64_t n_in, const int64_t *n_in_dev,
                                       const uint32_t *out_keys, int64_t n_out, const int64_t *n_out_dev,
                                       spc_pack_spec spec, spc_geom geom, int32_t t, uint32_t flags, void *buf,
                                       size_t buf_bytes, uint32_t *status, spc_kmap *kmap_out, void *stream) {
    if (spec.bits_b + spec.bits_x + spec.bits_y + spec.bits_z > 32)
        return fail(SPC_ERR_RANGE, "spc_build_kmap32: the pack spec needs more than 32 bits");
    return build_kmap(in_keys, n_in, n_in_dev, out_keys, n_out, n_out_dev, spec, geom, t, flags, buf, buf_bytes, status,
                      kmap_out, stream, 4);
}

namespace spc {
void kmap_defer_begin(void *scratch, size_t scratch_bytes, int64_t order_rows) {
    memset(&g_defer.b, 0, sizeof(g_defer.b));
    g_defer.max_kd = 0;
    g_defer.tiles = 0;
    g_defer.orders.clear();
    g_defer.order_rows = order_rows;
    g_defer.flushed = false;
    g_defer.batch_orders = false;
    g_defer.scratch = order_rows > 0 ? order_scratch(scratch, scratch_bytes, order_rows) : OrderScratch{};
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
    KmapBatch &b = g_defer.b;
    if (g_defer.batch_orders) {   // (an earlier, flushed batch may own the ordered maps)
        if (!g_defer.scratch.ok) return fail(SPC_ERR_WORKSPACE, "network kmaps: density-order scratch too small");
        b.ord_keys = g_defer.scratch.keys;
        b.ord_total = g_defer.scratch.total;
        b.ord_key_bits = ord_key_bits((int)g_defer.orders.size());
    }
    spc_status s = launch_kmaps(b, g_defer.max_kd, g_defer.tiles, st);
    if (s == SPC_OK) s = run_orders(g_defer.orders, g_defer.scratch, g_defer.order_rows, st);
    return s;
}
}  // namespace spc

// ------------------------------------------------------------------------------------
// multi-GPU range sharding of one scene: per shard the output range and its input halo
// ------------------------------------------------------------------------------------
namespace spc {
__global__ void k_shard_ranges(const uint64_t *__restrict__ in, int64_t n_in_cap, const int64_t *n_in_dev,
                               const uint64_t *__restrict__ out, int64_t n_out_cap, const int64_t *n_out_dev,
                               int64_t d_min, int64_t d_max, int n_shards, int64_t *__restrict__ bounds) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_shards) return;
    const int64_t n_in = dev_count(n_in_cap, n_in_dev), n_out = dev_count(n_out_cap, n_out_dev);
    const int64_t lo = n_out * r / n_shards, hi = n_out * (r + 1) / n_shards;
    int64_t ilo = 0, ihi = 0;
    if (hi > lo) {
        ilo = lower_bound_g<uint64_t>(in, n_in, out[lo] + (uint64_t)d_min);
        ihi = lower_bound_g<uint64_t>(in, n_in, out[hi - 1] + (uint64_t)d_max + 1ull);
    }
    bounds[4 * r] = lo;
    bounds[4 * r + 1] = hi;
    bounds[4 * r + 2] = ilo;
    bounds[4 * r + 3] = ihi > ilo ? ihi : ilo;
}
}  // namespace spc

extern "C" spc_status spc_shard_ranges(const uint64_t *in_keys, int64_t n_in, const int64_t *n_in_dev,
                                       const uint64_t *out_keys, int64_t n_out, const int64_t *n_out_dev,
                                       spc_pack_spec spec, spc_geom geom, int32_t n_shards, int64_t *bounds_dev,
                                       void *stream) {
    SPC_CHECK_ARG(n_shards >= 1 && bounds_dev && n_in >= 0 && n_out >= 0, "bad shard arguments");
    SPC_CHECK_ARG((in_keys || n_in == 0) && (out_keys || n_out == 0), "null keys");
    KmapPlan pl;
    spc_status s = make_plan(geom, SPC_T_ALL_OS, 0, pl);
    if (s != SPC_OK) return s;
    // extreme packed query offsets of the map: q + delta per axis with delta = e * spacing,
    // e in [lo, lo + K - 1] (a transposed map queries q - delta: negated and swapped)
    const int64_t w[3] = {1ll << (spec.bits_y + spec.bits_z), 1ll << spec.bits_z, 1};
    int64_t d_lo = 0, d_hi = 0;
    for (int a = 0; a < 3; ++a) {
        d_lo += (int64_t)pl.lo[a] * pl.spacing * w[a];
        d_hi += (int64_t)(pl.lo[a] + pl.kk[a] - 1) * pl.spacing * w[a];
    }
    if (geom.transposed) {
        const int64_t t0 = d_lo;
        d_lo = -d_hi;
        d_hi = -t0;
    }
    SPC_CUDA(launch_pdl(k_shard_ranges, dim3((n_shards + 127) / 128), dim3(128), 0, as_stream(stream), in_keys, n_in,
                        n_in_dev, out_keys, n_out, n_out_dev, d_lo, d_hi, (int)n_shards, bounds_dev));
    SPC_LAUNCH_CHECK("k_shard_ranges");
    return SPC_OK;
}

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
