// spc_sort.cu -- A1 pack, A2 sort-once, A3 grouped downsampling (Eq. 1 / Eq. 3).
//
// LSD radix sort over the USED key bits only (8-bit digits), onesweep style:
//   k_hist_all  : the digit histograms of EVERY pass in one read of the keys (k_pack
//                 computes them itself while packing, so spc_pack_sort skips this)
//   k_hist_scan : exclusive scans of those histograms (one CTA per pass)
//   k_onesweep  : one launch per pass: stable in-tile ranking, then the tile's global
//                 digit offsets by decoupled look-back over the preceding tiles, then a
//                 scatter staged through shared memory (coalesced digit runs)
// Every kernel reads the element count from device memory (n_dev), so the whole
// indexing phase runs without host syncs.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "spc_common.cuh"

namespace spc {

constexpr int SORT_THREADS = 256;
constexpr int SORT_ITEMS = 4;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;   // 1024 keys per tile
constexpr int SORT_WARPS = SORT_THREADS / 32;

// exclusive block scan of one int per thread (256 threads); returns the block total
__device__ __forceinline__ int block_excl_scan_256(int v, int *warp_sums, int &total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < SORT_WARPS ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < SORT_WARPS) warp_sums[lane] = s;   // inclusive
    }
    __syncthreads();
    int before = (w > 0 ? warp_sums[w - 1] : 0) + x - v;
    total = warp_sums[SORT_WARPS - 1];
    __syncthreads();
    return before;
}

// ---- onesweep LSD radix sort --------------------------------------------------------------
// k_hist_all   : digit histograms of EVERY pass in one read of the keys (smem, then global atomics)
// k_hist_scan  : exclusive scan of each pass's 256-bin histogram -> global digit bases
// k_onesweep   : one launch per pass; tiles are claimed in order from an atomic counter,
//                ranked locally (__match_any_sync, stable), and get their global offsets by
//                decoupled look-back over the per-tile digit counts of earlier tiles.
// keys per tile = SORT_THREADS * ITEMS, ITEMS in {2, 4, 8}: the smallest tiles that still
// give >= 2 tiles per SM's worth of CTAs, so small sorts (one scan, ~100k keys) spread
// over every SM instead of ~50 CTAs
constexpr int OS_ITEMS_MIN = 2;
constexpr int MAX_PASSES = 8;
constexpr uint32_t ST_AGG = 1u << 30, ST_INC = 2u << 30, ST_VAL = (1u << 30) - 1;

template <typename KeyT>
__global__ void __launch_bounds__(SORT_THREADS) k_hist_all(const KeyT *__restrict__ keys, int64_t n_cap,
                                                           const int64_t *n_dev, int passes,
                                                           unsigned int *__restrict__ ghist) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ unsigned int h[MAX_PASSES][256];
    for (int i = threadIdx.x; i < passes * 256; i += SORT_THREADS) h[i / 256][i % 256] = 0;
    __syncthreads();
    const int64_t n = dev_count(n_cap, n_dev);
    for (int64_t i = blockIdx.x * (int64_t)SORT_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * SORT_THREADS) {
        const KeyT k = keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += SORT_THREADS)
        if (h[i / 256][i % 256]) atomicAdd(&ghist[i], h[i / 256][i % 256]);
}

__global__ void k_hist_scan(unsigned int *__restrict__ ghist, int passes) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    // one warp per pass: exclusive scan of 256 counters in place
    const int p = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (p >= passes) return;
    unsigned int *h = ghist + p * 256;
    unsigned int carry = 0;
    for (int base = 0; base < 256; base += 32) {
        const unsigned int v = h[base + lane];
        unsigned int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        h[base + lane] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
}

template <typename KeyT, bool VALS, int OS_ITEMS>
__global__ void __launch_bounds__(SORT_THREADS) k_onesweep(const KeyT *__restrict__ keys_in,
                                                           const int32_t *__restrict__ vals_in, int64_t n_cap,
                                                           const int64_t *n_dev, int shift,
                                                           const unsigned int *__restrict__ gbase,
                                                           unsigned int *tile_status, unsigned int *tile_counter,
                                                           KeyT *__restrict__ keys_out,
                                                           int32_t *__restrict__ vals_out) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ int tile_s;
    __shared__ unsigned int excl_s[256];
    __shared__ int local_start[256];
    __shared__ int cnt[SORT_WARPS][256];
    __shared__ int warp_sums[SORT_WARPS];
    constexpr int OS_TILE = SORT_THREADS * OS_ITEMS;
    __shared__ KeyT skeys[OS_TILE];
    __shared__ int32_t svals[VALS ? OS_TILE : 1];

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t n = dev_count(n_cap, n_dev);
    if (tid == 0) tile_s = (int)atomicAdd(tile_counter, 1u);
#pragma unroll
    for (int ww = 0; ww < SORT_WARPS; ++ww) cnt[ww][tid] = 0;
    __syncthreads();
    const int tile = tile_s;
    const int64_t base = (int64_t)tile * OS_TILE;
    if (base >= n) return;
    const int tile_valid = (int)imin64(OS_TILE, n - base);

    KeyT key[OS_ITEMS];
    int32_t val[OS_ITEMS];
    int rank[OS_ITEMS];
    unsigned dig[OS_ITEMS];
#pragma unroll
    for (int r = 0; r < OS_ITEMS; ++r) {
        const int li = w * (32 * OS_ITEMS) + r * 32 + lane;   // warp-contiguous chunk: stable order
        const int64_t idx = base + li;
        const bool valid = li < tile_valid;
        key[r] = valid ? keys_in[idx] : (KeyT)~0ull;
        if (VALS) val[r] = valid ? (vals_in ? vals_in[idx] : (int32_t)idx) : 0;
        dig[r] = valid ? (unsigned)((key[r] >> shift) & 255u) : 256u + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, dig[r]);
        const int before = __popc(peers & lanemask_lt());
        const int c = valid ? cnt[w][dig[r]] : 0;
        rank[r] = c + before;
        __syncwarp();
        if (valid && before == 0) cnt[w][dig[r]] = c + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    int tile_cnt;
    {
        int s = 0;
#pragma unroll
        for (int ww = 0; ww < SORT_WARPS; ++ww) {
            const int c = cnt[ww][tid];
            cnt[ww][tid] = s;
            s += c;
        }
        tile_cnt = s;
        int tot;
        local_start[tid] = block_excl_scan_256(s, warp_sums, tot);
    }
    // ---- decoupled look-back: thread tid owns digit tid --------------------------------
    {
        unsigned int *st = tile_status + (int64_t)tile * 256 + tid;
        if (tile == 0) {
            atomicExch(st, ST_INC | (unsigned)tile_cnt);
            excl_s[tid] = 0;
        } else {
            atomicExch(st, ST_AGG | (unsigned)tile_cnt);
            // look back 8 predecessors per round trip (independent loads), newest first
            unsigned int excl = 0;
            int j = tile - 1;
            while (j >= 0) {
                unsigned int v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    v[q] = (j - q >= 0) ? *((const volatile unsigned int *)(tile_status + (int64_t)(j - q) * 256 + tid))
                                        : 0u;
                int consumed = 0;
                bool stop = false;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (j - q < 0 || (v[q] & ~ST_VAL) == 0) break;   // before tile 0 / not published yet
                    excl += v[q] & ST_VAL;
                    ++consumed;
                    if (v[q] & ST_INC) { stop = true; break; }
                }
                if (stop) break;
                j -= consumed;
            }
            atomicExch(st, ST_INC | (excl + (unsigned)tile_cnt));
            excl_s[tid] = excl;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < OS_ITEMS; ++r) {
        if (dig[r] < 256u) {
            const int lp = local_start[dig[r]] + cnt[w][dig[r]] + rank[r];
            skeys[lp] = key[r];
            if (VALS) svals[lp] = val[r];
        }
    }
    __syncthreads();
    for (int s = tid; s < tile_valid; s += SORT_THREADS) {
        const KeyT k = skeys[s];
        const int d = (int)((k >> shift) & 255u);
        const int64_t g = (int64_t)gbase[d] + excl_s[d] + (s - local_start[d]);
        keys_out[g] = k;
        if (VALS) vals_out[g] = svals[s];
    }
}

template <typename KeyT>
__global__ void k_copy_keys(const KeyT *__restrict__ a, int64_t n_cap, const int64_t *n_dev,
                            KeyT *__restrict__ b, const int32_t *vals_in, int32_t *vals_out) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    const int64_t n = dev_count(n_cap, n_dev);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        b[i] = a[i];
        if (vals_out) vals_out[i] = vals_in ? vals_in[i] : (int32_t)i;
    }
}

static int os_items(int64_t n) {
    for (int it = OS_ITEMS_MIN; it < 8; it *= 2)
        if ((n + SORT_THREADS * 2 * it - 1) / (SORT_THREADS * 2 * it) < 2 * num_sms()) return it;
    return 8;
}
static int os_tiles(int64_t n, int items) { return (int)((n + SORT_THREADS * items - 1) / (SORT_THREADS * items)); }

size_t radix_sort_workspace(int64_t n, bool with_vals) {
    Sizer s;
    const int nt = os_tiles(n > 0 ? n : 1, OS_ITEMS_MIN);
    s.take<unsigned int>((size_t)MAX_PASSES * 256);                 // histograms / bases
    s.take<unsigned int>((size_t)MAX_PASSES * (nt * 256 + 32));      // tile status + counters
    s.take<uint64_t>((size_t)n);
    if (with_vals) s.take<int32_t>((size_t)n);
    return s.used + 256;
}

template <typename KeyT>
static spc_status radix_sort_t(const KeyT *keys_in, const int32_t *vals_in, int64_t n, const int64_t *n_dev, int n_bits,
                               KeyT *keys_out, int32_t *vals_out, void *ws, size_t ws_bytes, cudaStream_t st,
                               bool hist_done) {
    if (n <= 0) return SPC_OK;
    const bool with_vals = vals_out != nullptr;
    const int passes = (n_bits + 7) / 8;
    if (passes > MAX_PASSES) return fail(SPC_ERR_INVALID_ARG, "radix_sort: too many key bits");
    Bump b(ws, ws_bytes);
    const int items = os_items(n);
    const int nt = os_tiles(n, items);
    unsigned int *hist = b.take<unsigned int>((size_t)MAX_PASSES * 256);
    const size_t stride = (size_t)nt * 256 + 32;
    // (the workspace holds the status of the smallest tiles; only the used part is cleared)
    unsigned int *status = b.take<unsigned int>((size_t)MAX_PASSES * ((size_t)os_tiles(n, OS_ITEMS_MIN) * 256 + 32));
    KeyT *ktmp = b.take<KeyT>((size_t)n);
    int32_t *vtmp = with_vals ? b.take<int32_t>((size_t)n) : nullptr;
    if (!b.ok()) return fail(SPC_ERR_WORKSPACE, "radix_sort: workspace too small");
    if (passes == 0) {
        SPC_CUDA(launch_pdl(k_copy_keys<KeyT>, dim3(256), dim3(256), 0, st, keys_in, n, n_dev, keys_out, vals_in, vals_out));
        SPC_LAUNCH_CHECK("k_copy_keys");
        return SPC_OK;
    }
    SPC_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned int) * passes * stride, st));
    if (!hist_done) {
        SPC_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned int) * MAX_PASSES * 256, st));
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>((n + 4095) / 4096, 2 * num_sms()));
        SPC_CUDA(launch_pdl(k_hist_all<KeyT>, dim3(g), dim3(SORT_THREADS), 0, st, keys_in, n, n_dev, passes, hist));
    }
    SPC_CUDA(launch_pdl(k_hist_scan, dim3(1), dim3(32 * MAX_PASSES), 0, st, hist, passes));
    SPC_LAUNCH_CHECK("radix histograms");
    const KeyT *src_k = keys_in;
    const int32_t *src_v = vals_in;
    for (int p = 0; p < passes; ++p) {
        const bool to_out = ((passes - 1 - p) % 2) == 0;
        KeyT *dst_k = to_out ? keys_out : ktmp;
        int32_t *dst_v = with_vals ? (to_out ? vals_out : vtmp) : nullptr;
        unsigned int *stp = status + (size_t)p * stride;
        unsigned int *ctr = stp + (size_t)nt * 256;
#define SPC_ONESWEEP(IT)                                                                                     \
    do {                                                                                                     \
        if (with_vals)                                                                                       \
            SPC_CUDA(launch_pdl(k_onesweep<KeyT, true, IT>, dim3(nt), dim3(SORT_THREADS), 0, st, src_k, src_v, n, n_dev, 8 * p, hist + p * 256, stp, \
                                                              ctr, dst_k, dst_v));                            \
        else                                                                                                 \
            SPC_CUDA(launch_pdl(k_onesweep<KeyT, false, IT>, dim3(nt), dim3(SORT_THREADS), 0, st, src_k, nullptr, n, n_dev, 8 * p, hist + p * 256,  \
                                                               stp, ctr, dst_k, nullptr));                    \
    } while (0)
        if (items == 2) SPC_ONESWEEP(2);
        else if (items == 4) SPC_ONESWEEP(4);
        else SPC_ONESWEEP(8);
#undef SPC_ONESWEEP
        SPC_LAUNCH_CHECK("onesweep pass");
        src_k = dst_k;
        src_v = dst_v;
    }
    return SPC_OK;
}

spc_status radix_sort(const uint64_t *keys_in, const int32_t *vals_in, int64_t n, const int64_t *n_dev, int n_bits,
                      uint64_t *keys_out, int32_t *vals_out, void *ws, size_t ws_bytes, cudaStream_t st,
                      bool hist_done) {
    return radix_sort_t(keys_in, vals_in, n, n_dev, n_bits, keys_out, vals_out, ws, ws_bytes, st, hist_done);
}
spc_status radix_sort(const uint32_t *keys_in, const int32_t *vals_in, int64_t n, const int64_t *n_dev, int n_bits,
                      uint32_t *keys_out, int32_t *vals_out, void *ws, size_t ws_bytes, cudaStream_t st,
                      bool hist_done) {
    return radix_sort_t(keys_in, vals_in, n, n_dev, n_bits, keys_out, vals_out, ws, ws_bytes, st, hist_done);
}

// ------------------------------------------------------------------------------------
// A1 pack + duplicate flag
// ------------------------------------------------------------------------------------
struct PackDev {
    int bb, bx, by, bz;
    int lo_room, hi_room;   // planned headroom below / above (reading A4): (out_stride-1)+reach / reach
};

template <typename KeyT>
__global__ void __launch_bounds__(256) k_pack(const int4 *__restrict__ coords, int64_t n_cap, const int64_t *n_dev, PackDev s,
                                              KeyT *__restrict__ keys, uint32_t *status, int passes,
                                              unsigned int *__restrict__ ghist) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ unsigned int h[MAX_PASSES][256];
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) h[i / 256][i % 256] = 0;
    __syncthreads();
    const int64_t n = dev_count(n_cap, n_dev);
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int4 c = coords[i];
        int64_t fb = c.x;
        int64_t fx = (int64_t)c.y + (1ll << (s.bx - 1));
        int64_t fy = (int64_t)c.z + (1ll << (s.by - 1));
        int64_t fz = (int64_t)c.w + (1ll << (s.bz - 1));
        // inside the field with the planned headroom on both sides, so downsampled
        // coordinates and kernel-map queries never carry or borrow into a neighbour field
        bool ok = fb >= 0 && fb < (1ll << s.bb) && fx >= s.lo_room && fx < (1ll << s.bx) - s.hi_room &&
                  fy >= s.lo_room && fy < (1ll << s.by) - s.hi_room && fz >= s.lo_room &&
                  fz < (1ll << s.bz) - s.hi_room;
        bad |= !ok;
        uint64_t k = ((uint64_t)fb << (s.bx + s.by + s.bz)) | ((uint64_t)fx << (s.by + s.bz)) |
                     ((uint64_t)fy << s.bz) | (uint64_t)fz;
        keys[i] = (KeyT)k;
        for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);   // sort histograms
    }
    if (__any_sync(0xffffffffu, bad) && status && (threadIdx.x & 31) == 0) atomicOr(status, SPC_FLAG_RANGE);
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x)
        if (h[i / 256][i % 256]) atomicAdd(&ghist[i], h[i / 256][i % 256]);
}

template <typename KeyT>
__global__ void k_flag_dups(const KeyT *__restrict__ keys, int64_t n_cap, const int64_t *n_dev,
                            uint32_t *status, uint32_t flag) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    const int64_t n = dev_count(n_cap, n_dev);
    bool dup = false;
    for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dup |= keys[i] <= keys[i - 1];
    if (__any_sync(0xffffffffu, dup) && (threadIdx.x & 31) == 0) atomicOr(status, flag);
}

__global__ void k_gather_rows(const char *__restrict__ src, int64_t ld_src, const int32_t *__restrict__ perm,
                              int64_t n_cap, const int64_t *n_dev, int row_bytes, char *__restrict__ dst,
                              int64_t ld_dst) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    const int64_t n = dev_count(n_cap, n_dev);
    const int vec = row_bytes / 16;
    const int64_t total = n * vec;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = t / vec;
        int v = (int)(t - r * vec);
        const int4 *s = reinterpret_cast<const int4 *>(src + (int64_t)perm[r] * ld_src) + v;
        int4 *d = reinterpret_cast<int4 *>(dst + r * ld_dst) + v;
        *d = __ldg(s);
    }
}

// ------------------------------------------------------------------------------------
// A3 grouped downsampling: tagged keys (level << used_bits) | (v0 & mask_level)
// ------------------------------------------------------------------------------------
struct LevelMasks {
    uint64_t mask[4];
};

__global__ void k_build_tagged(const uint64_t *__restrict__ v0, int64_t n_cap, const int64_t *n_dev, int L,
                               LevelMasks m, int used_bits, uint64_t *__restrict__ tagged,
                               int64_t *__restrict__ total_dev) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    const int64_t n = dev_count(n_cap, n_dev);
    if (blockIdx.x == 0 && threadIdx.x == 0) *total_dev = n * L;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * L; i += (int64_t)gridDim.x * blockDim.x) {
        int l = (int)(i / n);
        int64_t r = i - (int64_t)l * n;
        tagged[i] = ((uint64_t)l << used_bits) | (v0[r] & m.mask[l]);
    }
}

__global__ void __launch_bounds__(SORT_THREADS) k_unique_count(const uint64_t *__restrict__ k, const int64_t *total_dev,
                                                               int *__restrict__ tile_cnt) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ int ws[SORT_WARPS];
    const int64_t total = *total_dev;
    const int64_t base = (int64_t)blockIdx.x * SORT_TILE;
    int c = 0;
#pragma unroll
    for (int it = 0; it < SORT_ITEMS; ++it) {
        int64_t i = base + threadIdx.x * SORT_ITEMS + it;
        if (i < total) c += (i == 0 || k[i] != k[i - 1]);
    }
    int tot;
    block_excl_scan_256(c, ws, tot);
    if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
}

// single CTA: scan tile counts, then the unique-prefix at each level boundary l*n
__global__ void __launch_bounds__(1024) k_unique_scan(int *__restrict__ tile_cnt, int n_tiles,
                                                      const uint64_t *__restrict__ k, const int64_t *total_dev,
                                                      int64_t n_cap, const int64_t *n_dev, int L,
                                                      int64_t *__restrict__ level_base, int64_t *__restrict__ level_n) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ int wsum[32];
    __shared__ int carry_s;
    __shared__ int red[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < n_tiles; base += 1024) {
        int i = base + threadIdx.x;
        int v = i < n_tiles ? tile_cnt[i] : 0;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            int s = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;
        }
        __syncthreads();
        int carry = carry_s;
        if (i < n_tiles) tile_cnt[i] = carry + (w > 0 ? wsum[w - 1] : 0) + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry_s = carry + wsum[31];
        __syncthreads();
    }
    const int64_t total_unique = carry_s;
    const int64_t n = dev_count(n_cap, n_dev);
    const int64_t total = *total_dev;
    for (int l = 0; l <= L; ++l) {
        int64_t b = (int64_t)l * n;
        int64_t pref;
        if (b >= total) {
            pref = total_unique;
        } else {
            int64_t tb = b / SORT_TILE;
            int c = 0;
            for (int64_t i = tb * SORT_TILE + threadIdx.x; i < b; i += 1024) c += (i == 0 || k[i] != k[i - 1]);
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if (lane == 0) red[w] = c;
            __syncthreads();
            if (threadIdx.x == 0) {
                int s = 0;
                for (int q = 0; q < 32; ++q) s += red[q];
                red[0] = s;
            }
            __syncthreads();
            pref = (int64_t)tile_cnt[tb] + red[0];
            __syncthreads();
        }
        if (threadIdx.x == 0) level_base[l] = pref;
    }
    __syncthreads();
    if (threadIdx.x < L) level_n[threadIdx.x] = level_base[threadIdx.x + 1] - level_base[threadIdx.x];
}

__global__ void __launch_bounds__(SORT_THREADS) k_unique_write(const uint64_t *__restrict__ k, const int64_t *total_dev,
                                                               int64_t n_cap, const int64_t *n_dev,
                                                               const int *__restrict__ tile_scan,
                                                               const int64_t *__restrict__ level_base,
                                                               uint64_t strip_mask, uint64_t *__restrict__ out,
                                                               int64_t out_stride) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ int ws[SORT_WARPS];
    const int64_t total = *total_dev;
    const int64_t n = dev_count(n_cap, n_dev);
    const int64_t base = (int64_t)blockIdx.x * SORT_TILE;
    if (base >= total) return;
    int f[SORT_ITEMS];
    int c = 0;
#pragma unroll
    for (int it = 0; it < SORT_ITEMS; ++it) {
        int64_t i = base + threadIdx.x * SORT_ITEMS + it;
        f[it] = (i < total) && (i == 0 || k[i] != k[i - 1]);
        c += f[it];
    }
    int tot;
    int pos = block_excl_scan_256(c, ws, tot) + tile_scan[blockIdx.x];
#pragma unroll
    for (int it = 0; it < SORT_ITEMS; ++it) {
        int64_t i = base + threadIdx.x * SORT_ITEMS + it;
        if (f[it]) {
            int l = (int)(i / n);
            out[(int64_t)l * out_stride + (pos - level_base[l])] = k[i] & strip_mask;
            ++pos;
        }
    }
}

// ------------------------------------------------------------------------------------
// NEXT-2 voxelization front-end (§2.1 v = floor(p / g); S:132 averaging):
// quantise + pack + histograms in one pass, the stable radix sort, then one pass that
// writes the unique keys, each voxel's first sorted position and the point -> voxel map,
// and a warp-per-voxel mean of the features in ascending point order
// ------------------------------------------------------------------------------------
struct VoxGrid {
    float g[3];
};

__global__ void __launch_bounds__(256) k_voxel_pack(const float *__restrict__ pts, int64_t ld,
                                                    const int32_t *__restrict__ batch, int64_t n_cap,
                                                    const int64_t *n_dev, VoxGrid vg, PackDev s,
                                                    uint64_t *__restrict__ keys, uint32_t *status,
                                                    unsigned long long *bad_point, int passes,
                                                    unsigned int *__restrict__ ghist, int64_t *total_out) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ unsigned int h[MAX_PASSES][256];
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) h[i / 256][i % 256] = 0;
    __syncthreads();
    const int64_t n = dev_count(n_cap, n_dev);
    if (blockIdx.x == 0 && threadIdx.x == 0) *total_out = n;
    bool out_of_field = false, non_finite = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v[3];
        bool fin = true;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            // float32 quotient, IEEE round-to-nearest (reading V1); a non-finite p gives a
            // non-finite quotient, so checking q covers both
            const float q = __fdiv_rn(pts[i * ld + d], vg.g[d]);
            const float f = floorf(q);
            const bool ok = isfinite(q) && f >= -2147483648.0f && f < 2147483648.0f;
            fin &= ok;
            v[d] = ok ? (int64_t)f : 0;
        }
        if (!fin) {
            non_finite = true;
            if (bad_point) atomicMin(bad_point, (unsigned long long)i);
        }
        const int64_t fb = batch ? batch[i] : 0;
        const int64_t fx = v[0] + (1ll << (s.bx - 1)), fy = v[1] + (1ll << (s.by - 1)), fz = v[2] + (1ll << (s.bz - 1));
        const bool ok = fb >= 0 && fb < (1ll << s.bb) && fx >= s.lo_room && fx < (1ll << s.bx) - s.hi_room &&
                        fy >= s.lo_room && fy < (1ll << s.by) - s.hi_room && fz >= s.lo_room &&
                        fz < (1ll << s.bz) - s.hi_room;
        out_of_field |= !ok;
        const uint64_t k = ((uint64_t)fb << (s.bx + s.by + s.bz)) | ((uint64_t)fx << (s.by + s.bz)) |
                           ((uint64_t)fy << s.bz) | (uint64_t)fz;
        keys[i] = k;
        for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);   // sort histograms
    }
    const bool r = __any_sync(0xffffffffu, out_of_field), f = __any_sync(0xffffffffu, non_finite);
    if (status && (threadIdx.x & 31) == 0 && (r || f))
        atomicOr(status, (r ? SPC_FLAG_RANGE : 0u) | (f ? SPC_FLAG_NONFINITE : 0u));
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x)
        if (h[i / 256][i % 256]) atomicAdd(&ghist[i], h[i / 256][i % 256]);
}

// unique keys, each voxel's first sorted position, and point -> voxel (a voxel's index is
// the number of run heads before it: the tile prefix from k_unique_scan + a block scan)
__global__ void __launch_bounds__(SORT_THREADS) k_voxel_segments(const uint64_t *__restrict__ k,
                                                                 const int32_t *__restrict__ perm,
                                                                 const int64_t *total_dev,
                                                                 const int *__restrict__ tile_scan,
                                                                 uint64_t *__restrict__ keys_out,
                                                                 int32_t *__restrict__ seg_start,
                                                                 int32_t *__restrict__ point_voxel) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    __shared__ int ws[SORT_WARPS];
    const int64_t total = *total_dev;
    const int64_t base = (int64_t)blockIdx.x * SORT_TILE;
    if (base >= total) return;
    int f[SORT_ITEMS];
    int c = 0;
#pragma unroll
    for (int it = 0; it < SORT_ITEMS; ++it) {
        const int64_t i = base + threadIdx.x * SORT_ITEMS + it;
        f[it] = (i < total) && (i == 0 || k[i] != k[i - 1]);
        c += f[it];
    }
    int tot;
    int pos = block_excl_scan_256(c, ws, tot) + tile_scan[blockIdx.x];
#pragma unroll
    for (int it = 0; it < SORT_ITEMS; ++it) {
        const int64_t i = base + threadIdx.x * SORT_ITEMS + it;
        if (i >= total) break;
        if (f[it]) {
            keys_out[pos] = k[i];
            seg_start[pos] = (int32_t)i;
            ++pos;
        }
        if (point_voxel) point_voxel[perm[i]] = pos - 1;
    }
}

// one warp per voxel, lane = channel: the fp32 sum of the voxel's points in ascending
// point index (stable sort order), divided by the count, rounded once to the output
__global__ void __launch_bounds__(256) k_voxel_mean(const float *__restrict__ feats, int64_t ld_f, int c,
                                                    const int32_t *__restrict__ perm,
                                                    const int32_t *__restrict__ seg_start, const int64_t *n_vox_dev,
                                                    const int64_t *total_dev, void *__restrict__ out, int64_t ld_out,
                                                    int out_dtype, int64_t *bad_point) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    if (bad_point && blockIdx.x == 0 && threadIdx.x == 0 && *bad_point == INT64_MAX) *bad_point = -1;
    if (c == 0) return;
    const int64_t nv = *n_vox_dev, total = *total_dev;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = w0; v < nv; v += nw) {
        const int64_t s = seg_start[v], e = v + 1 < nv ? seg_start[v + 1] : total;
        const float cnt = (float)(e - s);
        for (int ch = lane; ch < c; ch += 32) {
            float acc = 0.f;
            for (int64_t j = s; j < e; ++j) acc = __fadd_rn(acc, feats[(int64_t)perm[j] * ld_f + ch]);
            const float m = __fdiv_rn(acc, cnt);
            if (out_dtype == SPC_F32) static_cast<float *>(out)[v * ld_out + ch] = m;
            else static_cast<__nv_bfloat16 *>(out)[v * ld_out + ch] = __float2bfloat16_rn(m);
        }
    }
}

__global__ void k_voxel_init(int64_t *bad_point, int64_t *n_vox, int64_t n_cap) {
    pdl_wait();
    pdl_trigger();
    if (bad_point) *bad_point = n_cap > 0 ? INT64_MAX : -1;
    if (n_vox && n_cap == 0) *n_vox = 0;
}

// ------------------------------------------------------------------------------------
// NEXT-3 spconv "regular" output sites: candidates p - delta on the coarse lattice (packed
// arithmetic; lattice test = the Eq. (1) mask leaves the key unchanged),
// compacted with one warp reservation, then the stable radix sort + unique
// ------------------------------------------------------------------------------------
struct BoxDeltas {
    int64_t d[SPC_MAX_KVOL];   // packed delta_k
};

__global__ void __launch_bounds__(256) k_regular_candidates(const uint64_t *__restrict__ in, int64_t n_cap,
                                                            const int64_t *n_dev, int kv, BoxDeltas bd,
                                                            uint64_t off_lattice, uint64_t *__restrict__ cand,
                                                            unsigned long long *count) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger();
    const int64_t n = dev_count(n_cap, n_dev);
    const int lane = threadIdx.x & 31;
    const int64_t total = n * kv;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // whole warps iterate together (ballot reservation)
    for (int64_t e0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31); e0 < total;
         e0 += stride) {
        const int64_t e = e0 + lane;
        bool keep = false;
        uint64_t c = 0;
        if (e < total) {
            const int64_t i = e / kv;
            const int k = (int)(e - i * kv);
            c = in[i] - (uint64_t)bd.d[k];   // packed(p) - packed(delta) = packed(p - delta)
            keep = (c & off_lattice) == 0;   // every spatial field a multiple of the out stride
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        unsigned long long base = 0;
        if (lane == 0 && bal) base = atomicAdd(count, (unsigned long long)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) cand[base + __popc(bal & lanemask_lt())] = c;
    }
}

}  // namespace spc

using namespace spc;

extern "C" size_t spc_pack_sort_workspace_size(int64_t n) {
    if (n < 0) n = 0;
    return align_up(sizeof(uint64_t) * (size_t)n, 256) + radix_sort_workspace(n, true) + 256;
}

namespace spc {
// pack + sort for 64-bit keys, or 32-bit keys when the spec's fields total <= 32 bits (the
// paper's default single-scan packing)
template <typename KeyT>
static spc_status pack_sort_t(const int32_t *coords, int64_t n, const int64_t *n_dev, spc_pack_spec spec, KeyT *keys_out,
                              int32_t *perm_out, uint32_t *status, void *ws, size_t ws_bytes, void *stream) {
    SPC_CHECK_ARG(n >= 0, "n < 0");
    if (n == 0) return SPC_OK;
    SPC_CHECK_ARG(coords && keys_out, "null coords/keys_out");
    SPC_CHECK_ARG(n < (int64_t)INT32_MAX, "n too large for int32 indices");
    const int used = spec.bits_b + spec.bits_x + spec.bits_y + spec.bits_z;
    SPC_CHECK_ARG(spec.bits_b >= 0 && spec.bits_x >= 2 && spec.bits_y >= 2 && spec.bits_z >= 2 && used <= 62,
                  "bad pack spec");
    if (used > (int)(8 * sizeof(KeyT)))
        return fail(SPC_ERR_RANGE, "spc_pack_sort32: the pack spec needs " + std::to_string(used) + " bits > 32");
    SPC_CHECK_ARG(spec.reach >= 0 && spec.out_stride >= 1 && (spec.out_stride & (spec.out_stride - 1)) == 0,
                  "pack spec: reach must be >= 0 and out_stride a power of two >= 1");
    if (ws_bytes < spc_pack_sort_workspace_size(n)) return fail(SPC_ERR_WORKSPACE, "spc_pack_sort: ws too small");
    cudaStream_t st = as_stream(stream);
    Bump b(ws, ws_bytes);
    KeyT *raw = b.take<KeyT>((size_t)n);
    void *rws = b.base + align_up(b.used, 256);
    size_t rws_bytes = ws_bytes - align_up(b.used, 256);
    PackDev pd{spec.bits_b, spec.bits_x, spec.bits_y, spec.bits_z, spec.out_stride - 1 + spec.reach, spec.reach};
    int grid = (int)imin64((n + 2047) / 2048, 2 * 148);
    // pack + all radix histograms in one pass over the coordinates (the histogram block is
    // the first region of the radix workspace)
    unsigned int *hist = reinterpret_cast<unsigned int *>(rws);   // == radix_sort's first workspace block
    SPC_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned int) * MAX_PASSES * 256, st));
    SPC_CUDA(launch_pdl(k_pack<KeyT>, dim3(grid), dim3(256), 0, st, reinterpret_cast<const int4 *>(coords), n, n_dev, pd,
                        raw, status, (used + 7) / 8, hist));
    SPC_LAUNCH_CHECK("k_pack");
    spc_status s = radix_sort(raw, nullptr, n, n_dev, used, keys_out, perm_out, rws, rws_bytes, st, true);
    if (s != SPC_OK) return s;
    if (status) {
        SPC_CUDA(launch_pdl(k_flag_dups<KeyT>, dim3(grid), dim3(256), 0, st, keys_out, n, n_dev, status, SPC_FLAG_DUPLICATE));
        SPC_LAUNCH_CHECK("k_flag_dups");
    }
    return SPC_OK;
}

// SPC_KMAP_CHECK_SORTED: flag keys that are not strictly ascending
spc_status flag_unsorted(const void *keys, int key_bytes, int64_t n_cap, const int64_t *n_dev, uint32_t *status,
                         cudaStream_t st) {
    if (key_bytes == 4)
        SPC_CUDA(launch_pdl(k_flag_dups<uint32_t>, dim3(64), dim3(256), 0, st, static_cast<const uint32_t *>(keys), n_cap,
                            n_dev, status, SPC_FLAG_UNSORTED));
    else
        SPC_CUDA(launch_pdl(k_flag_dups<uint64_t>, dim3(64), dim3(256), 0, st, static_cast<const uint64_t *>(keys), n_cap,
                            n_dev, status, SPC_FLAG_UNSORTED));
    SPC_LAUNCH_CHECK("k_flag_dups");
    return SPC_OK;
}
}  // namespace spc

extern "C" spc_status spc_pack_sort(const int32_t *coords, int64_t n, const int64_t *n_dev, spc_pack_spec spec,
                                    uint64_t *keys_out, int32_t *perm_out, uint32_t *status, void *ws, size_t ws_bytes,
                                    void *stream) {
    return pack_sort_t(coords, n, n_dev, spec, keys_out, perm_out, status, ws, ws_bytes, stream);
}

extern "C" spc_status spc_pack_sort32(const int32_t *coords, int64_t n, const int64_t *n_dev, spc_pack_spec spec,
                                      uint32_t *keys_out, int32_t *perm_out, uint32_t *status, void *ws, size_t ws_bytes,
                                      void *stream) {
    return pack_sort_t(coords, n, n_dev, spec, keys_out, perm_out, status, ws, ws_bytes, stream);
}

extern "C" spc_status spc_gather_rows(const void *src, int64_t ld_src_bytes, const int32_t *perm, int64_t n,
                                      const int64_t *n_dev, int32_t row_bytes, void *dst, int64_t ld_dst_bytes,
                                      void *stream) {
    SPC_CHECK_ARG(n >= 0, "n < 0");
    if (n == 0) return SPC_OK;
    SPC_CHECK_ARG(src && perm && dst, "null pointer");
    SPC_CHECK_ARG(row_bytes > 0 && row_bytes % 16 == 0 && ld_src_bytes % 16 == 0 && ld_dst_bytes % 16 == 0 &&
                      ((uintptr_t)src % 16) == 0 && ((uintptr_t)dst % 16) == 0,
                  "rows must be 16-byte aligned multiples of 16 bytes");
    int64_t work = n * (row_bytes / 16);
    int grid = (int)imin64((work + 255) / 256, 8 * 148);
    SPC_CUDA(launch_pdl(k_gather_rows, dim3(grid), dim3(256), 0, as_stream(stream), (const char *)src, ld_src_bytes, perm, n, n_dev, row_bytes,
                                                      (char *)dst, ld_dst_bytes));
    SPC_LAUNCH_CHECK("k_gather_rows");
    return SPC_OK;
}

extern "C" size_t spc_downsample_workspace_size(int64_t n, int32_t n_levels) {
    if (n < 0) n = 0;
    int64_t tot = n * (n_levels > 0 ? n_levels : 1);
    Sizer s;
    s.take<uint64_t>((size_t)tot);       // tagged
    s.take<uint64_t>((size_t)tot);       // sorted tagged
    s.take<int64_t>(8);                  // total, level_base
    s.take<int>((size_t)(tot / SORT_TILE + 2));
    return s.used + radix_sort_workspace(tot, false) + 512;
}

extern "C" spc_status spc_downsample(const uint64_t *keys, int64_t n, const int64_t *n_dev, spc_pack_spec spec,
                                     int32_t n_levels, const int32_t *log2_stride_host, uint64_t *level_keys,
                                     int64_t *level_n_dev, void *ws, size_t ws_bytes, void *stream) {
    SPC_CHECK_ARG(n >= 0 && n_levels >= 1 && n_levels <= 4, "n < 0 or n_levels not in 1..4");
    SPC_CHECK_ARG(log2_stride_host && level_keys && level_n_dev && (keys || n == 0), "null pointer");
    const int minb = min(spec.bits_x, min(spec.bits_y, spec.bits_z));
    LevelMasks lm{};
    for (int l = 0; l < n_levels; ++l) {
        int m = log2_stride_host[l];
        if (m < 0 || m > minb - 1)
            return fail(SPC_ERR_INVALID_ARG, "spc_downsample: log2 stride " + std::to_string(m) + " out of range");
        if ((1ll << m) > spec.out_stride)
            return fail(SPC_ERR_RANGE, "spc_downsample: stride " + std::to_string(1ll << m) +
                                           " exceeds the planned spec.out_stride " + std::to_string(spec.out_stride));
        lm.mask[l] = spc_downsample_mask(spec, m);
    }
    if (ws_bytes < spc_downsample_workspace_size(n, n_levels))
        return fail(SPC_ERR_WORKSPACE, "spc_downsample: ws too small");
    cudaStream_t st = as_stream(stream);
    if (n == 0) {
        SPC_CUDA(cudaMemsetAsync(level_n_dev, 0, sizeof(int64_t) * n_levels, st));
        return SPC_OK;
    }
    const int used = spec.bits_b + spec.bits_x + spec.bits_y + spec.bits_z;
    const int64_t tot = n * n_levels;
    Bump b(ws, ws_bytes);
    uint64_t *tagged = b.take<uint64_t>((size_t)tot);
    uint64_t *sorted = b.take<uint64_t>((size_t)tot);
    int64_t *scal = b.take<int64_t>(8);   // [0] total, [1..5] level_base
    const int nt = (int)((tot + SORT_TILE - 1) / SORT_TILE);
    int *tile_cnt = b.take<int>((size_t)(tot / SORT_TILE + 2));
    void *rws = b.base + align_up(b.used, 256);
    size_t rws_bytes = ws_bytes - align_up(b.used, 256);
    int grid = (int)imin64((tot + 255) / 256, 8 * 148);
    SPC_CUDA(launch_pdl(k_build_tagged, dim3(grid), dim3(256), 0, st, keys, n, n_dev, n_levels, lm, used, tagged, scal));
    SPC_LAUNCH_CHECK("k_build_tagged");
    const int tag_bits = n_levels > 2 ? 2 : (n_levels > 1 ? 1 : 0);
    spc_status s = radix_sort(tagged, nullptr, tot, scal, used + tag_bits, sorted, nullptr, rws, rws_bytes, st, false);
    if (s != SPC_OK) return s;
    SPC_CUDA(launch_pdl(k_unique_count, dim3(nt), dim3(SORT_THREADS), 0, st, sorted, scal, tile_cnt));
    SPC_CUDA(launch_pdl(k_unique_scan, dim3(1), dim3(1024), 0, st, tile_cnt, nt, sorted, scal, n, n_dev, n_levels, scal + 1, level_n_dev));
    const uint64_t strip = used >= 64 ? ~0ull : ((1ull << used) - 1);
    SPC_CUDA(launch_pdl(k_unique_write, dim3(nt), dim3(SORT_THREADS), 0, st, sorted, scal, n, n_dev, tile_cnt, scal + 1, strip, level_keys, n));
    SPC_LAUNCH_CHECK("unique");
    return SPC_OK;
}

// ------------------------------------------------------------------------------------
// NEXT-2 voxelization front-end (spc.h)
// ------------------------------------------------------------------------------------
extern "C" size_t spc_voxelize_workspace_size(int64_t n) {
    if (n < 0) n = 0;
    Sizer z;
    z.take<uint64_t>((size_t)n);                        // raw keys
    z.take<uint64_t>((size_t)n);                        // sorted keys
    z.take<int32_t>((size_t)n);                         // perm
    z.take<int32_t>((size_t)n);                         // seg_start
    z.take<int64_t>(4);                                 // total, level_base[2]
    z.take<int>((size_t)(n / SORT_TILE + 2));           // tile counts
    return z.used + radix_sort_workspace(n, true) + 512;
}

extern "C" spc_status spc_voxelize(const float *points, int64_t ld, const int32_t *batch, int64_t n, const int64_t *n_dev,
                                   const float *grid_host, spc_pack_spec spec, const float *feats, int64_t ld_feats,
                                   int32_t c, uint64_t *keys_out, int64_t *n_vox_dev, int32_t *point_voxel,
                                   void *feats_out, int64_t ld_out, int32_t out_dtype, uint32_t *status,
                                   int64_t *bad_point_dev, void *ws, size_t ws_bytes, void *stream) {
    SPC_CHECK_ARG(n >= 0 && n < (int64_t)INT32_MAX, "n out of range");
    SPC_CHECK_ARG(grid_host && n_vox_dev && (keys_out || n == 0), "null grid / keys_out / n_vox_dev");
    for (int d = 0; d < 3; ++d)
        SPC_CHECK_ARG(std::isfinite(grid_host[d]) && grid_host[d] > 0.f, "grid sizes must be finite and > 0");
    SPC_CHECK_ARG(c >= 0 && (c == 0 || (feats && feats_out && ld_feats >= c && ld_out >= c)),
                  "c < 0, or features without feats / feats_out / row strides >= c");
    SPC_CHECK_ARG(out_dtype == SPC_F32 || out_dtype == SPC_BF16, "out_dtype must be SPC_F32 or SPC_BF16");
    const int used = spec.bits_b + spec.bits_x + spec.bits_y + spec.bits_z;
    SPC_CHECK_ARG(spec.bits_b >= 0 && spec.bits_x >= 2 && spec.bits_y >= 2 && spec.bits_z >= 2 && used <= 62,
                  "bad pack spec");
    SPC_CHECK_ARG(spec.reach >= 0 && spec.out_stride >= 1 && (spec.out_stride & (spec.out_stride - 1)) == 0,
                  "pack spec: reach must be >= 0 and out_stride a power of two >= 1");
    cudaStream_t st = as_stream(stream);
    if (n == 0) {
        SPC_CUDA(launch_pdl(k_voxel_init, dim3(1), dim3(1), 0, st, bad_point_dev, n_vox_dev, (int64_t)0));
        SPC_LAUNCH_CHECK("k_voxel_init");
        return SPC_OK;
    }
    SPC_CHECK_ARG(points && ld >= 3, "null points or ld < 3");
    if (ws_bytes < spc_voxelize_workspace_size(n)) return fail(SPC_ERR_WORKSPACE, "spc_voxelize: ws too small");
    Bump b(ws, ws_bytes);
    uint64_t *raw = b.take<uint64_t>((size_t)n);
    uint64_t *sorted = b.take<uint64_t>((size_t)n);
    int32_t *perm = b.take<int32_t>((size_t)n);
    int32_t *seg = b.take<int32_t>((size_t)n);
    int64_t *scal = b.take<int64_t>(4);
    const int nt = (int)((n + SORT_TILE - 1) / SORT_TILE);
    int *tile_cnt = b.take<int>((size_t)(n / SORT_TILE + 2));
    void *rws = b.base + align_up(b.used, 256);
    const size_t rws_bytes = ws_bytes - align_up(b.used, 256);
    unsigned int *hist = reinterpret_cast<unsigned int *>(rws);   // == radix_sort's first workspace block
    SPC_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned int) * MAX_PASSES * 256, st));
    SPC_CUDA(launch_pdl(k_voxel_init, dim3(1), dim3(1), 0, st, bad_point_dev, (int64_t *)nullptr, n));
    VoxGrid vg{{grid_host[0], grid_host[1], grid_host[2]}};
    PackDev pd{spec.bits_b, spec.bits_x, spec.bits_y, spec.bits_z, spec.out_stride - 1 + spec.reach, spec.reach};
    const int grid = (int)imin64((n + 2047) / 2048, 2 * 148);
    SPC_CUDA(launch_pdl(k_voxel_pack, dim3(grid), dim3(256), 0, st, points, ld, batch, n, n_dev, vg, pd, raw, status,
                        reinterpret_cast<unsigned long long *>(bad_point_dev), (used + 7) / 8, hist, scal));
    SPC_LAUNCH_CHECK("k_voxel_pack");
    spc_status s = radix_sort(raw, nullptr, n, n_dev, used, sorted, perm, rws, rws_bytes, st, true);
    if (s != SPC_OK) return s;
    SPC_CUDA(launch_pdl(k_unique_count, dim3(nt), dim3(SORT_THREADS), 0, st, sorted, scal, tile_cnt));
    SPC_CUDA(launch_pdl(k_unique_scan, dim3(1), dim3(1024), 0, st, tile_cnt, nt, sorted, scal, n, n_dev, 1, scal + 1,
                        n_vox_dev));
    SPC_CUDA(launch_pdl(k_voxel_segments, dim3(nt), dim3(SORT_THREADS), 0, st, sorted, perm, scal, tile_cnt, keys_out,
                        seg, point_voxel));
    SPC_LAUNCH_CHECK("k_voxel_segments");
    const int mgrid = (int)imin64((n + 7) / 8, 16 * 148);
    SPC_CUDA(launch_pdl(k_voxel_mean, dim3(mgrid), dim3(256), 0, st, feats, ld_feats, (int)c, perm, seg, n_vox_dev, scal,
                        feats_out, ld_out, (int)out_dtype, bad_point_dev));
    SPC_LAUNCH_CHECK("k_voxel_mean");
    return SPC_OK;
}

// ------------------------------------------------------------------------------------
// NEXT-3 regular output sites (spc.h)
// ------------------------------------------------------------------------------------
static int64_t geom_kvol(const spc_geom &g) {
    const int ky = g.kernel_size_y > 0 ? g.kernel_size_y : g.kernel_size;
    const int kz = g.kernel_size_z > 0 ? g.kernel_size_z : g.kernel_size;
    return (int64_t)g.kernel_size * ky * kz;
}

extern "C" size_t spc_regular_outputs_workspace_size(int64_t n_in, spc_geom geom) {
    if (n_in < 0) n_in = 0;
    const int64_t cap = n_in * std::max<int64_t>(1, geom_kvol(geom));
    Sizer z;
    z.take<uint64_t>((size_t)cap);
    z.take<uint64_t>((size_t)cap);
    z.take<int64_t>(4);
    z.take<int>((size_t)(cap / SORT_TILE + 2));
    return z.used + radix_sort_workspace(cap, false) + 512;
}

extern "C" spc_status spc_regular_outputs(const uint64_t *in_keys, int64_t n_in, const int64_t *n_in_dev,
                                          spc_pack_spec spec, spc_geom geom, uint64_t *out_keys, int64_t *n_out_dev,
                                          void *ws, size_t ws_bytes, void *stream) {
    SPC_CHECK_ARG(n_in >= 0 && n_out_dev && (n_in == 0 || (in_keys && out_keys)), "null pointer or n_in < 0");
    const int ks[3] = {geom.kernel_size, geom.kernel_size_y > 0 ? geom.kernel_size_y : geom.kernel_size,
                       geom.kernel_size_z > 0 ? geom.kernel_size_z : geom.kernel_size};
    for (int a = 0; a < 3; ++a)
        SPC_CHECK_ARG(ks[a] >= 1 && ks[a] <= 5, "kernel sizes must be in 1..5");
    SPC_CHECK_ARG(!geom.transposed && geom.stride >= 1 && geom.dilation >= 1 && geom.tensor_stride >= 1,
                  "a forward (non-transposed) geometry with stride, dilation, tensor_stride >= 1");
    const int64_t out_stride = (int64_t)geom.tensor_stride * geom.stride;
    SPC_CHECK_ARG((out_stride & (out_stride - 1)) == 0, "tensor_stride * stride must be a power of two");
    const int64_t spacing = (int64_t)geom.tensor_stride * geom.dilation;
    int lo[3], reach_units = 0;
    for (int a = 0; a < 3; ++a) {
        lo[a] = ks[a] % 2 ? -(ks[a] - 1) / 2 : 0;
        reach_units = std::max(reach_units, std::max(-lo[a], lo[a] + ks[a] - 1));
    }
    if (reach_units * spacing > spec.reach)
        return fail(SPC_ERR_RANGE, "spc_regular_outputs: kernel reach " + std::to_string(reach_units * spacing) +
                                       " exceeds the planned spec.reach = " + std::to_string(spec.reach));
    if (out_stride > spec.out_stride)
        return fail(SPC_ERR_RANGE, "spc_regular_outputs: output stride exceeds the planned spec.out_stride");
    const int kv = ks[0] * ks[1] * ks[2];
    if (ws_bytes < spc_regular_outputs_workspace_size(n_in, geom))
        return fail(SPC_ERR_WORKSPACE, "spc_regular_outputs: ws too small");
    cudaStream_t st = as_stream(stream);
    if (n_in == 0) {
        SPC_CUDA(cudaMemsetAsync(n_out_dev, 0, sizeof(int64_t), st));
        return SPC_OK;
    }
    BoxDeltas bd{};
    int k = 0;
    for (int ex = lo[0]; ex < lo[0] + ks[0]; ++ex)
        for (int ey = lo[1]; ey < lo[1] + ks[1]; ++ey)
            for (int ez = lo[2]; ez < lo[2] + ks[2]; ++ez)
                bd.d[k++] = spc_pack_offset(spec, (int32_t)(ex * spacing), (int32_t)(ey * spacing), (int32_t)(ez * spacing));
    int m = 0;
    while ((1ll << m) < out_stride) ++m;
    const int used = spec.bits_b + spec.bits_x + spec.bits_y + spec.bits_z;
    const uint64_t spatial = ((1ull << (spec.bits_x + spec.bits_y + spec.bits_z)) - 1);
    const uint64_t off_lattice = spatial & ~spc_downsample_mask(spec, m);   // low m bits of each spatial field
    const int64_t cap = n_in * kv;
    Bump b(ws, ws_bytes);
    uint64_t *cand = b.take<uint64_t>((size_t)cap);
    uint64_t *sorted = b.take<uint64_t>((size_t)cap);
    int64_t *scal = b.take<int64_t>(4);   // [0] candidate count, [1..2] unique prefix
    const int nt = (int)((cap + SORT_TILE - 1) / SORT_TILE);
    int *tile_cnt = b.take<int>((size_t)(cap / SORT_TILE + 2));
    void *rws = b.base + align_up(b.used, 256);
    const size_t rws_bytes = ws_bytes - align_up(b.used, 256);
    SPC_CUDA(cudaMemsetAsync(scal, 0, sizeof(int64_t), st));
    const int grid = (int)imin64((cap + 255) / 256, 8 * 148);
    SPC_CUDA(launch_pdl(k_regular_candidates, dim3(grid), dim3(256), 0, st, in_keys, n_in, n_in_dev, kv, bd, off_lattice,
                        cand, reinterpret_cast<unsigned long long *>(scal)));
    SPC_LAUNCH_CHECK("k_regular_candidates");
    spc_status s = radix_sort(cand, nullptr, cap, scal, used, sorted, nullptr, rws, rws_bytes, st, false);
    if (s != SPC_OK) return s;
    SPC_CUDA(launch_pdl(k_unique_count, dim3(nt), dim3(SORT_THREADS), 0, st, sorted, scal, tile_cnt));
    SPC_CUDA(launch_pdl(k_unique_scan, dim3(1), dim3(1024), 0, st, tile_cnt, nt, sorted, scal, cap, scal, 1, scal + 1,
                        n_out_dev));
    SPC_CUDA(launch_pdl(k_unique_write, dim3(nt), dim3(SORT_THREADS), 0, st, sorted, scal, cap, scal, tile_cnt, scal + 1,
                        ~0ull, out_keys, cap));
    SPC_LAUNCH_CHECK("regular outputs unique");
    return SPC_OK;
}
