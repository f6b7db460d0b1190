/*
 * spc.h -- C ABI of libspc, the B200 (sm_100a) sparse-convolution hot path of
 * "Accelerating Sparse Convolutions in Voxel-Based Point Cloud Networks" (Spira,
 * arXiv 2511.20834).  Citations "P:N" are lines of that paper's PAPER.md.
 *
 * Conventions (all entry points)
 * ------------------------------
 * - Pointers are DEVICE pointers unless the name ends in _host.  No torch types.
 * - `stream` is a cudaStream_t passed as void*.  Every call only ENQUEUES work on it
 *   and returns without a device synchronisation; none of them allocates device
 *   memory: persistent buffers and scratch ("ws") come from the caller.
 * - Host-detectable errors return a status != SPC_OK immediately (nothing enqueued);
 *   spc_last_error_detail() names the offending argument.  Data-dependent errors are
 *   OR-ed by the kernels into a caller-owned device uint32 status word (SPC_FLAG_*),
 *   readable after the caller synchronises the stream.
 * - Sizes: every function that consumes a data-dependent count takes the host
 *   CAPACITY (n_*) and an optional device pointer to the actual count (n_*_dev, may be
 *   NULL = the capacity is the count).  This keeps whole network passes free of host
 *   syncs and CUDA-graph capturable.
 * - Index spaces: voxel i of a coordinate set is its position in the SORTED key array
 *   (canonical lexicographic order).
 * - Weights: user layout [K^3][C_in][C_out], offset index k in lexicographic (dx,dy,dz)
 *   order with dz fastest (k of -delta = K^3-1-k).
 * - Kernels are compiled for sm_100a only.  There is no CPU fallback.
 */
#ifndef SPC_H
#define SPC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPC_VERSION 4

typedef enum {
    SPC_OK = 0,
    SPC_ERR_INVALID_ARG = 1,   /* null pointer, negative size, bad dtype/shape/alignment */
    SPC_ERR_UNSUPPORTED = 2,   /* even K, channels not a multiple of 16, ...            */
    SPC_ERR_RANGE = 3,         /* coordinate extent does not fit the key fields          */
    SPC_ERR_DUPLICATE = 4,
    SPC_ERR_UNSORTED = 5,
    SPC_ERR_CAPACITY = 6,
    SPC_ERR_WORKSPACE = 7,     /* ws smaller than *_workspace_size()                     */
    SPC_ERR_CUDA = 8           /* a CUDA runtime call failed (detail has the message)    */
} spc_status;

/* device status word bits (set by kernels with atomicOr) */
#define SPC_FLAG_RANGE 0x1u      /* pack: coordinate outside its key field            */
#define SPC_FLAG_DUPLICATE 0x2u  /* pack_sort: two equal keys                         */
#define SPC_FLAG_UNSORTED 0x4u   /* build_kmap (SPC_KMAP_CHECK_SORTED): input unsorted */
#define SPC_FLAG_CAPACITY 0x8u   /* a device count exceeded its host capacity          */
#define SPC_FLAG_NONFINITE 0x10u /* voxelize: a point coordinate (or p/g) is not finite  */

typedef enum { SPC_F32 = 0, SPC_F16 = 1, SPC_BF16 = 2 } spc_dtype;

const char *spc_status_string(int status);
const char *spc_last_error_detail(void);   /* thread-local, last failing call */
int spc_version(void);
size_t spc_kmap_struct_bytes(void);        /* sizeof(spc_kmap), for binding layout checks */

/* Process-wide tuning options of the feature computation (performance only: every
 * value gives the same Eq. (2) result).  Read by later spc_conv_forward calls; not
 * thread-safe against concurrent calls.  value < 0 restores the default.
 * Returns SPC_ERR_INVALID_ARG for an unknown option. */
typedef enum {
    SPC_OPT_CONV_TILE_ROWS = 0,   /* 0 = device heuristic (default); 128 / 256 force the OS/WS tile rows */
    SPC_OPT_CONV_STAGE_KB = 1,    /* pipeline stage size cap in KB (default 72; 256-wide pairs 48)*/
    SPC_OPT_CONV_OS_SPLIT = 2,    /* 1 (default): small OS launches split a tile's offsets over CTAs */
    SPC_OPT_CONV_SPLIT_MIN = 3,   /* minimum offsets per split part (default 2)                   */
    SPC_OPT_CONV_CLAIM_AHEAD = 4, /* dynamic tile claims ahead of the gather warps, 1..3 (default 1) */
    SPC_OPT_CONV_DENSITY_ORDER = 5, /* 1 (default): use a map's density-ordered OS table if it has one */
    SPC_OPT_PDL = 6,              /* 1 (default): programmatic dependent launches               */
    SPC_OPT_KMAP_POOL_KEYS = 7,   /* test hook: shared window pool of the z-delta build in keys
                                   * (default 4096; smaller forces the global-memory fallback)    */
    SPC_OPT_CONV_DENSE_CENTRE = 8, /* 1: the centre of an all-WS submanifold map runs as a dense
                                   * TMA-fed GEMM that initialises the accumulator (default 0)    */
    SPC_OPT_CONV_CTA_PAIR = 9,    /* CTA pairs (cta_group::2, M = 256) for outputs >= 192 wide:
                                   * 0 off, 1 auto (default), 2 wherever the shape allows       */
    SPC_OPT_CONV_MAPS_READY = 10, /* 1: the caller asserts that the kernel map and the prepared
                                   * weights of the next spc_conv_forward calls were complete
                                   * before the preceding kernel of their stream STARTED (true
                                   * for every layer but the first of a network pass): the
                                   * kernel then decodes tiles and streams weights while that
                                   * kernel drains (programmatic dependent launch) (default 0)  */
    SPC_OPT_CONV_BULK_RED = 11,   /* 1 (default): the weight-stationary scatter reduces 64-column
                                   * row segments with bulk reductions (TMA); 0: red.global.add */
    SPC_OPT_WGRAD_ITEMS_PER_SM = 12, /* spc_conv_wgrad work items per SM over the map's pair
                                   * capacity (default 16: smaller items balance better)       */
    SPC_OPT_CONV_SPLIT_TILES = 13, /* an OS launch splits its tiles' offsets over CTAs when
                                   * 2 x (tiles x N-tiles) <= this (default 0: the SM count) */
    SPC_OPT_CONV_MAX_CTAS = 14,   /* > 0: the persistent feature kernels use at most this many
                                   * CTAs (one per SM), leaving SMs to a concurrent stream     */
    SPC_OPT_CONV_BLK_KB = 15,     /* OS gather-index blocks: two in flight (the next tile's loads
                                   * while this tile gathers) up to this many KB for both, beside
                                   * a ring of >= 2 stages (default 128; 64: K = 5 keeps one)    */
    SPC_OPT_COUNT = 16
} spc_option;
spc_status spc_set_option(int32_t option, int64_t value);
int64_t spc_get_option(int32_t option);

/* Device-side event trace of the feature kernels (observability; off by default).
 * buf: device uint64 [1 + 2*cap]; buf[0] counts records (the caller zeroes it), record i
 * = (buf[1+2i] = %globaltimer ns, buf[2+2i] = launch << 48 | event << 40 | cta << 24 | aux).
 * Events: 0 CTA entry, 1 after the PDL wait, 2 setup done, 3 tile record published,
 * 4 first stage of a tile full, 5 tile's MMAs committed, 6 tile's epilogue done, 7 CTA
 * exit (aux = tile sequence number of the CTA where it applies).  Launches are numbered
 * from 0 after every spc_set_trace call; spc_trace_launch_desc(launch) names one.
 * buf = NULL turns tracing off.  Captured CUDA graphs keep the buffer they saw. */
spc_status spc_set_trace(void *buf, int64_t cap);
const char *spc_trace_launch_desc(int32_t launch);

/* ================================================================================
 * A1  Packed keys (§5.3)
 *
 * key = b << (Bx+By+Bz) | (x + 2^(Bx-1)) << (By+Bz) | (y + 2^(By-1)) << Bz | (z + 2^(Bz-1))
 *
 * z is least significant, x most significant among the spatial fields; the
 * batch index b (unsigned, never offset or masked) sits above x (reading A5).
 * Each spatial field is biased by 2^(B-1), a multiple of every stride 2^m with
 * m <= B-1, so AND-masking the biased field equals floor rounding of the signed
 * coordinate (reading A3) and packed(q) + packed(delta) = packed(q + delta)
 * as long as q + delta stays inside the field (headroom, reading A4).
 * Bb + Bx + By + Bz <= 62 (two bits are reserved for the level tag of spc_downsample).
 * ================================================================================ */
typedef struct {
    int32_t bits_b, bits_x, bits_y, bits_z;
    /* headroom the field widths were planned for (reading A4): every packed
     * coordinate v must satisfy  -2^(B-1) + (out_stride-1) + reach <= v <= 2^(B-1)-1 - reach
     * per axis (spc_pack_sort flags SPC_FLAG_RANGE otherwise), so downsampling up to
     * stride out_stride and queries q +- delta with |delta| <= reach per axis never
     * carry or borrow across fields.  spc_downsample refuses strides > out_stride and
     * spc_build_kmap / spc_network_kmaps refuse maps whose reach r*tensor_stride*dilation
     * exceeds `reach` (SPC_ERR_RANGE): no silent truncation. */
    int32_t reach;       /* >= 0                                                       */
    int32_t out_stride;  /* >= 1, a power of two                                       */
} spc_pack_spec;

/* Smallest field widths such that every coordinate in [lo_host, hi_host] (per axis),
 * every output of downsampling up to stride max_out_stride (rounding moves a
 * coordinate down by at most max_out_stride-1) and every query q +- delta with
 * |delta| <= max_reach stays inside its biased field (reading A4/A6).  The planned
 * max_reach / max_out_stride are recorded in the spec (reach, out_stride).
 * Returns SPC_ERR_RANGE (detail names the axis and the bits required) if the total
 * exceeds 62 bits. */
spc_status spc_plan_pack(const int32_t lo_host[3], const int32_t hi_host[3], int32_t n_batch,
                         int32_t max_out_stride, int32_t max_reach, spc_pack_spec *out_host);

/* packed(delta) = dx*2^(By+Bz) + dy*2^Bz + dz as a signed 64-bit word. */
int64_t spc_pack_offset(spc_pack_spec spec, int32_t dx, int32_t dy, int32_t dz);

/* The downsample mask of P:327-336 for s_q = 2^m: per spatial field B-m ones then m
 * zeros; the batch field all ones (read as bitwise AND, reading A1). */
uint64_t spc_downsample_mask(spc_pack_spec spec, int32_t m);

/* ================================================================================
 * A1+A2  spc_pack_sort -- pack int32 coordinates and sort them once
 *
 * coords   : int32 [n][4] rows (b, x, y, z), any row order.  n is the capacity; n_dev
 *            (nullable) the live row count on the device (rows [0, *n_dev) are packed and
 *            sorted), so a whole pass stays graph-capturable for any scan size <= n.
 * keys_out : uint64 [n], ascending (stable LSD radix sort over the used key bits).
 * perm_out : int32 [n] (nullable): keys_out[p] = key(coords[perm_out[p]]).  The caller
 *            gathers feature rows with it (spc_gather_rows).
 * status   : device uint32, OR-ed with SPC_FLAG_RANGE (a coordinate does not fit its
 *            field with the planned headroom spec.reach / spec.out_stride; its key is
 *            undefined if it does not fit the field at all) and SPC_FLAG_DUPLICATE (two
 *            rows with equal coordinates).
 * ws       : >= spc_pack_sort_workspace_size(n) bytes.
 * ================================================================================ */
size_t spc_pack_sort_workspace_size(int64_t n);
spc_status spc_pack_sort(const int32_t *coords, int64_t n, const int64_t *n_dev, spc_pack_spec spec, uint64_t *keys_out,
                         int32_t *perm_out, uint32_t *status, void *ws, size_t ws_bytes, void *stream);

/* 32-bit keys (NEXT-1 ablation): the same pack + sort when bits_b+x+y+z <= 32 (e.g. one
 * scan at 12/12/8); SPC_ERR_RANGE otherwise.  Same workspace size. */
spc_status spc_pack_sort32(const int32_t *coords, int64_t n, const int64_t *n_dev, spc_pack_spec spec,
                           uint32_t *keys_out, int32_t *perm_out, uint32_t *status, void *ws, size_t ws_bytes,
                           void *stream);

/* ================================================================================
 * NEXT-2  spc_voxelize -- the voxelization front-end fused with pack + sort
 *         (§2.1 v = floor(p_raw / g); SPEC S:70-78 quantize, S:132 averaging)
 *
 * points  : float32 rows, point i at points[i*ld + 0..2] = (x, y, z) in metres.  n is
 *           the capacity, n_dev (nullable) the live point count on the device.
 * batch   : int32 [n] batch index per point (nullable: 0).
 * grid    : host float[3], g > 0.  v = floor(p / g) per axis with the quotient rounded
 *           to float32 (IEEE round-to-nearest division; reading V1), floor
 *           toward -infinity.
 * spec    : pack spec for the voxel coordinates (spc_plan_pack over the expected voxel
 *           range); a voxel outside its field with the planned headroom sets
 *           SPC_FLAG_RANGE as in spc_pack_sort.
 * feats   : float32 rows feats[i*ld_feats + 0..c) (nullable when c == 0).
 * keys_out: uint64 [n]: the n_vox sorted unique voxel keys (A1 layout) first -- the same
 *           keys spc_pack_sort would give for the voxel coordinates, ready for
 *           spc_downsample / spc_build_kmap.
 * n_vox_dev   : device int64, the voxel count.
 * point_voxel : int32 [n] (nullable): index in keys_out of point i's voxel.
 * feats_out   : [n][ld_out] rows of out_dtype (SPC_F32 or SPC_BF16; nullable when c == 0):
 *           row v = the mean of the features of voxel v's points, summed in fp32 in
 *           ascending point index (the sort is stable), divided by the count, rounded once.
 * status  : device uint32 (nullable), OR-ed with SPC_FLAG_NONFINITE (a coordinate or its
 *           quotient is not finite or leaves int32) and SPC_FLAG_RANGE; outputs are
 *           undefined when a flag is set.
 * bad_point_dev : device int64 (nullable): the smallest index of a non-finite point, or
 *           -1 when there is none (the S:73 diagnostic, on the device).
 * ws      : >= spc_voxelize_workspace_size(n) bytes, stream-ordered scratch.
 * ================================================================================ */
size_t spc_voxelize_workspace_size(int64_t n);
spc_status spc_voxelize(const float *points, int64_t ld, const int32_t *batch, int64_t n, const int64_t *n_dev,
                        const float *grid_host, spc_pack_spec spec, const float *feats, int64_t ld_feats, int32_t c,
                        uint64_t *keys_out, int64_t *n_vox_dev, int32_t *point_voxel, void *feats_out, int64_t ld_out,
                        int32_t out_dtype, uint32_t *status, int64_t *bad_point_dev, void *ws, size_t ws_bytes,
                        void *stream);

/* dst row r = src row perm[r] (row_bytes each, 16-byte aligned rows).  n_dev nullable. */
spc_status spc_gather_rows(const void *src, int64_t ld_src_bytes, const int32_t *perm, int64_t n,
                           const int64_t *n_dev, int32_t row_bytes, void *dst, int64_t ld_dst_bytes,
                           void *stream);

/* ================================================================================
 * A3  spc_downsample -- Eq. (1) for several output strides at once, each computed
 *     directly from V_0 (Eq. (3)):  V_m = unique(sort(V_0 & mask_m)).
 *
 * The AND mask is not monotone across fields, so every level is re-sorted (reading A2).
 * All levels go through ONE radix sort of n_levels*n tagged keys and one unique
 * compaction (the grouped phase 1 of network-wide indexing).
 *
 * keys      : sorted unique V_0 keys, capacity n (n_dev: actual count, nullable).
 * log2_stride_host[l] : m_l in 1..min(B)-1 (output stride 2^m_l).  n_levels <= 4.
 * level_keys: device buffer [n_levels][n]; level l's sorted unique keys are written at
 *             level_keys + l*n.
 * level_n_dev: device int64 [n_levels], the unique counts.
 * ================================================================================ */
size_t spc_downsample_workspace_size(int64_t n, int32_t n_levels);
spc_status spc_downsample(const uint64_t *keys, int64_t n, const int64_t *n_dev, spc_pack_spec spec,
                          int32_t n_levels, const int32_t *log2_stride_host, uint64_t *level_keys,
                          int64_t *level_n_dev, void *ws, size_t ws_bytes, void *stream);

/* ================================================================================
 * A4-A8  Kernel maps (§2.2, z-delta search P:253-301 §5.2, layouts P:393-421)
 * ================================================================================ */
typedef struct {
    int32_t kernel_size;   /* K (x size of the offset box; odd K: Delta(K, s_p)) */
    int32_t stride;        /* layer stride s_l: 1 = submanifold (V_q = V_p), 2 = down/up */
    int32_t dilation;      /* d >= 1 (offsets delta * d; not in the paper, reading A11)  */
    int32_t tensor_stride; /* stride of the FINE coordinate set (s_p of a normal layer,  */
                           /* s_q of a transposed one); offsets are spaced by           */
                           /* tensor_stride * dilation (Delta(K, s_p))           */
    int32_t transposed;    /* 0: out = V_{ts*stride} (coarse) or V_ts (submanifold), in = V_ts */
                           /* 1: out = V_ts (fine), in = V_{ts*stride} (coarse); triple  */
                           /*    (k,i,j) iff in_j = out_i - delta_k  (reading A8)        */
    /* a non-cubic box (Kx = kernel_size, Ky, Kz; 0 = kernel_size).  Every
     * size is in 1..5; per axis the offsets are e*spacing with e in {-(K-1)/2 .. (K-1)/2}
     * for odd K and e in {0 .. K-1} for even K (reading E1: the K = 2 down/up layers'
     * {0, s_p}^3).  Weight offsets k are lexicographic (e_x, e_y, e_z), e_z fastest.
     * SPC_KMAP_HALVE_SYMMETRIC applies to centred boxes (every size odd) only and is
     * ignored otherwise; the map's reach is max |e| * spacing over the box. */
    int32_t kernel_size_y;
    int32_t kernel_size_z;
} spc_geom;

/* NEXT-3  spconv's "regular" output rule for a forward layer of box `geom` (odd sizes
 * centred, i.e. spconv padding (K-1)/2; even sizes {0..K-1}): the sorted unique sites
 *   V_out = { p - delta : p in V_in, delta in the box (spacing tensor_stride*dilation),
 *             every spatial coordinate a multiple of tensor_stride*stride }
 * -- every output site whose kernel footprint touches an input (for K = 2, stride 2 this
 * is Eq. (1)'s V_q).  in_keys: sorted unique keys (n_in_dev nullable).  out_keys: room for
 * n_in * Kx*Ky*Kz keys; n_out_dev: device int64 count.  The map between V_in and V_out is
 * then an ordinary spc_build_kmap(in_keys, out_keys, ..., geom).  SPC_ERR_RANGE when the
 * box reach or the output stride exceeds the spec's planned headroom. */
size_t spc_regular_outputs_workspace_size(int64_t n_in, spc_geom geom);
spc_status spc_regular_outputs(const uint64_t *in_keys, int64_t n_in, const int64_t *n_in_dev, spc_pack_spec spec,
                               spc_geom geom, uint64_t *out_keys, int64_t *n_out_dev, void *ws, size_t ws_bytes,
                               void *stream);

/* dataflow threshold t: offset k is dense (output-stationary) iff
 * L1(e_k) < t, where e_k in {-r..r}^3 is the offset in units of tensor_stride*dilation
 * (reading A15).  t = 0: all weight-stationary; t >= 3r+1 (SPC_T_ALL_OS): all OS. */
#define SPC_T_ALL_OS (-1)
#define SPC_T_ALL_WS 0

#define SPC_KMAP_HALVE_SYMMETRIC 0x1u /* submanifold: store WS pairs of k < centre only;
                                       * needs in_keys == out_keys (else SPC_ERR_INVALID_ARG)   */
#define SPC_KMAP_CHECK_SORTED 0x2u    /* debug: flag unsorted / duplicate input keys          */
#define SPC_KMAP_COUNT_SEARCHES 0x4u  /* debug: count binary searches and scan probes        */
#define SPC_KMAP_DENSITY_ORDER 0x8u   /* OS part: also build a density-ordered copy of the OS
                                       * table (outputs stably sorted by their match mask) that
                                       * spc_conv_forward uses: tiles of outputs with similar
                                       * neighbour patterns skip more empty offset chunks     */
#define SPC_KMAP_SIMPLE_BSEARCH 0x10u /* ablation: build the OS table with the
                                       * paper's "Simple BSearch" baseline:
                                       * one global binary search per (output, offset) =
                                       * |V_q|*K^3 searches instead of |V_q|*K^2 (z-delta).
                                       * Needs an all-OS t (SPC_ERR_UNSUPPORTED otherwise);
                                       * DENSITY_ORDER is ignored; standalone builds only.   */

#define SPC_MAX_KVOL 125

/* A built kernel map: plain struct of device pointers into one caller buffer.
 * OS part : os_table[i*k_dense + c] = input index of output i at dense offset
 *           dense_k[c], or -1 (unfiltered |V_q| x K_dense layout).
 * WS part : list l (offset list_k[l]) holds counts_dev[list_k[l]] pairs
 *           ws_pairs[(l*n_out + p)*2 + {0,1}] = (in j, out i), no sentinels, in no
 *           particular order (reading A16).  With halving, list_mirror[l] != 0 means
 *           the pair also stands for (in i, out j) at offset K^3-1-list_k[l].
 * counts_dev: int32 [2*SPC_MAX_KVOL].  counts_dev[k] = matches found for offset k (the
 *           K^3 auxiliary buffer; offsets skipped by halving read 0 -- their count
 *           equals that of K^3-1-k by symmetry); counts_dev[SPC_MAX_KVOL + l] = pairs
 *           stored in WS list l.
 * tile_mask_dev (OS): bit c of word [tile*words + c/32] set iff some output of the
 *           128-row tile has a match at dense offset c (empty chunks are skipped).
 * os_rows / os_table_ord / tile_mask_ord (SPC_KMAP_DENSITY_ORDER, else NULL): the OS
 *           table with its rows permuted (row p holds output os_rows[p]; outputs stably
 *           sorted by a direction key: bit j set iff the output matches offset k or its
 *           mirror K^3-1-k, j = rank of the pair among the dense pairs (submanifold centre
 *           skipped), folded onto 16 bits (16 - ceil(log2 #ordered maps) in a network
 *           build)) and the tile masks of that order.  Same values as os_table, other row
 *           order; the feature computation writes row p's result to output os_rows[p]. */
typedef struct {
    spc_geom geom;
    int32_t t;            /* effective threshold (SPC_T_ALL_OS resolved)            */
    int32_t k_vol;        /* K^3                                                    */
    int32_t k_dense;      /* number of dense offsets (OS part)                      */
    int32_t n_lists;      /* number of stored WS lists                              */
    int32_t halved;       /* 1 if SPC_KMAP_HALVE_SYMMETRIC was applied              */
    int32_t key_bits;     /* 64, or 32 for maps built by spc_build_kmap32 (in_keys /
                           * out_keys then point to uint32 keys)                    */
    int32_t tile_words;   /* 32-bit words per OS tile in tile_mask_dev              */
    int64_t n_in;         /* capacities (host)                                      */
    int64_t n_out;
    const int64_t *n_in_dev;   /* actual counts (device, nullable)                  */
    const int64_t *n_out_dev;
    const uint64_t *in_keys;
    const uint64_t *out_keys;
    int32_t *os_table;
    int32_t *ws_pairs;
    int32_t *counts_dev;
    uint32_t *tile_mask_dev;
    unsigned long long *search_stats_dev; /* [2]: binary searches, scan probes (or NULL) */
    int32_t *os_rows;        /* [n_out] density order -> output index (or NULL)     */
    int32_t *os_table_ord;   /* [n_out * k_dense] OS table in density order          */
    uint32_t *tile_mask_ord; /* tile masks of the density order                      */
    int32_t *tile_order;     /* density order: 128-row tiles by descending weight (popcount
                              * of the tile mask), then 256-row tiles likewise; then the
                              * weights in those two orders ([4][ceil(n_out/128)])           */
    int16_t dense_k[SPC_MAX_KVOL];
    int16_t list_k[SPC_MAX_KVOL];
    int8_t list_mirror[SPC_MAX_KVOL];
} spc_kmap;

/* bytes of the caller buffer spc_build_kmap needs for this geometry/t/capacities */
size_t spc_kmap_bytes(spc_geom geom, int32_t t, uint32_t flags, int64_t n_in, int64_t n_out);

/* Build the kernel map of one layer with the one-shot z-delta search:
 * per (output i, offset group g) one lower_bound of q_i + packed(delta_anchor(g)) in
 * the sorted input keys, then a forward cursor scan for the group's other members in
 * ascending query order.  Both layouts are written straight from the search (OS block
 * staged per 128-output tile, WS pairs compacted with warp-aggregated atomics): there
 * is no separate transpose / filter post-processing pass.
 * in_keys/out_keys: sorted unique keys of the input/output coordinate sets (the same
 * array for a submanifold layer).  buf: >= spc_kmap_bytes() bytes, 256-byte aligned.
 * status: device uint32 (nullable) for SPC_FLAG_UNSORTED / SPC_FLAG_CAPACITY.
 * kmap_out_host: filled with pointers into buf.
 * Returns SPC_ERR_RANGE if the map's reach r*tensor_stride*dilation exceeds spec.reach
 * or its coarse stride tensor_stride*stride exceeds spec.out_stride (reading A4). */
spc_status spc_build_kmap(const uint64_t *in_keys, int64_t n_in, const int64_t *n_in_dev,
                          const uint64_t *out_keys, int64_t n_out, const int64_t *n_out_dev,
                          spc_pack_spec spec, spc_geom geom, int32_t t, uint32_t flags, void *buf,
                          size_t buf_bytes, uint32_t *status, spc_kmap *kmap_out_host, void *stream);

/* NEXT-1 ablation (the paper packs one scan into 32 bits, 12/12/8):
 * the same build over uint32 keys from spc_pack_sort32.  The spec's fields must total
 * <= 32 bits (SPC_ERR_RANGE otherwise); network-wide builds and SPC_KMAP_SIMPLE_BSEARCH
 * stay 64-bit (SPC_ERR_UNSUPPORTED).  The map is used by spc_conv_forward unchanged. */
spc_status spc_build_kmap32(const uint32_t *in_keys, int64_t n_in, const int64_t *n_in_dev,
                            const uint32_t *out_keys, int64_t n_out, const int64_t *n_out_dev,
                            spc_pack_spec spec, spc_geom geom, int32_t t, uint32_t flags, void *buf,
                            size_t buf_bytes, uint32_t *status, spc_kmap *kmap_out_host, void *stream);

/* Export the map as (k, out, in) int32 triples sorted lexicographically (parity
 * tooling; [sync]: synchronises `stream`).  Returns the nnz in *nnz_host; writes at
 * most cap triples to triples_host (host memory). */
spc_status spc_kmap_export(const spc_kmap *kmap, int32_t *triples_host, int64_t cap, int64_t *nnz_host,
                           void *stream);

/* ================================================================================
 * A9-A12  spc_conv_forward -- Eq. (2) with the output-stationary part (dense offsets)
 * and the weight-stationary part (sparse offsets) of the map.
 *
 * f_in   : [n_in][ld_in] elements of in_dtype, first c_in used.  Rows 16-byte aligned.
 * weight : prepared weights (spc_prepare_weight) for this (K^3, c_in, c_out, in_dtype).
 * f_out  : [n_out][ld_out] elements of out_dtype, first c_out written.
 * residual: nullable, [n_out][ld_res] elements of out_dtype, added to the result.
 * Arithmetic: f16/bf16 inputs -> tcgen05.mma kind::f16 with fp32 accumulation in TMEM;
 * f32 inputs -> FFMA (fp32).  c_in, c_out multiples of 16 (f16/bf16); f32: c_in % 4 == 0,
 * c_out % 8 == 0;
 * c_out <= 256 per weight tile (larger c_out is tiled).
 * ws     : >= spc_conv_workspace_size() bytes: the fp32 accumulator of the WS part and of
 *          split output tiles (small levels: a tile's offsets are split over CTAs, the
 *          last arriving CTA finishes the tile), followed by tile arrival counters.
 *          CONTRACT: ws must be all-zero before its first use (cudaMemset once); every
 *          call returns it to all-zero, so it can be reused by any later call of any
 *          shape without clearing.  One ws per stream (calls sharing a ws must be
 *          stream-ordered).  ws may be NULL only for maps without a WS part; then no
 *          tile is split.
 * Tile geometry (128/256-row tiles, split factor) is chosen on the device from the live
 * row count *n_out_dev, so capacity-sized network maps need no host sync.
 * ================================================================================ */
size_t spc_prepared_weight_bytes(int32_t k_vol, int32_t c_in, int32_t c_out, int32_t in_dtype);
spc_status spc_prepare_weight(const void *weight, int32_t k_vol, int32_t c_in, int32_t c_out,
                              int32_t in_dtype, void *prepared, void *stream);
size_t spc_conv_workspace_size(const spc_kmap *kmap, int32_t c_out, int32_t out_dtype);
spc_status spc_conv_forward(const spc_kmap *kmap, const void *f_in, int64_t ld_in, int32_t in_dtype,
                            int32_t c_in, const void *weight, int32_t c_out, void *f_out,
                            int64_t ld_out, int32_t out_dtype, const void *residual, int64_t ld_res,
                            void *ws, size_t ws_bytes, void *stream);

/* ================================================================================
 * fused epilogue, training path (beyond the paper's inference scope,
 * S:15; the gradients of Eq. (2), §2.1).
 *
 * spc_epilogue: applied to every FINAL output element (column c) of spc_conv_forward_ex,
 * in the order of the networks' residual blocks (relu(bn(conv(x)) + shortcut)):
 *     y = acc * scale[c] + shift[c];  y += residual (if any);  if (relu) y = max(y, 0).
 * scale / shift: device fp32 [c_out], 16-byte aligned, each nullable (identity).
 * spc_conv_forward(...) == spc_conv_forward_ex(..., epi = NULL, ...).
 *
 * spc_bn_fold: inference batch norm folded on the device:
 *     scale = gamma / sqrt(var + eps),  shift = beta - mean * scale   (fp32 [c]).
 * ================================================================================ */
typedef struct {
    const float *scale;
    const float *shift;
    int32_t relu;
} spc_epilogue;
spc_status spc_conv_forward_ex(const spc_kmap *kmap, const void *f_in, int64_t ld_in, int32_t in_dtype,
                               int32_t c_in, const void *weight, int32_t c_out, void *f_out,
                               int64_t ld_out, int32_t out_dtype, const void *residual, int64_t ld_res,
                               const spc_epilogue *epi, void *ws, size_t ws_bytes, void *stream);
spc_status spc_bn_fold(const float *gamma, const float *beta, const float *mean, const float *var, float eps,
                       int32_t c, float *scale, float *shift, void *stream);

/* Weight preparation for the data gradient.  dF_in[j] = sum over the map's matches
 * (i, j, k) of dF_out[i] W_k^T is Eq. (2) run backwards; it reuses the forward kernels:
 *  - submanifold layer (centred box): the SAME map (by symmetry (j,i,k) in M <=> (i,j,
 *    K^3-1-k) in M) with weights W'_k = W_{K^3-1-k}^T  -> SPC_WEIGHT_DGRAD_MIRROR;
 *  - strided layer: the transposed map (out = the layer's inputs, in = its outputs, same
 *    k, spc_geom.transposed = 1) with W'_k = W_k^T            -> SPC_WEIGHT_DGRAD;
 *  - transposed layer: the strided map, W'_k = W_k^T           -> SPC_WEIGHT_DGRAD.
 * Then spc_conv_forward(dgrad map, dF_out, c_in = layer c_out, prepared W', c_out = layer
 * c_in, dF_in); gradients of inputs read by several layers accumulate through the
 * residual operand (residual == f_out is allowed: every element is read, then written, by
 * the same thread).  weight: [k_vol][c_in][c_out] of the FORWARD layer; the prepared weight
 * is that of a (k_vol, c_out -> c_in) layer.  (SPC_WEIGHT_FORWARD = spc_prepare_weight.) */
typedef enum { SPC_WEIGHT_FORWARD = 0, SPC_WEIGHT_DGRAD = 1, SPC_WEIGHT_DGRAD_MIRROR = 2 } spc_weight_mode;
spc_status spc_prepare_weight_ex(const void *weight, int32_t k_vol, int32_t c_in, int32_t c_out,
                                 int32_t in_dtype, int32_t mode, void *prepared, void *stream);

/* spc_conv_wgrad -- dW_k[c][o] += sum over the map's pairs (j, i) at offset k of
 *                   F_in[j][c] * dF_out[i][o]   for every k (the weight gradient of Eq. (2)).
 * kmap   : the FORWARD layer's map, any t (dense columns: pairs (os_table[i][c], i),
 *          sentinel rows contribute nothing, empty 128-row tiles skipped; WS lists;
 *          halved lists also contribute their mirrored pairs to K^3-1-k).
 * f_in   : [n_in][ld_in] forward inputs; d_out: [n_out][ld_dout] output gradients (both
 *          in_dtype, rows 16-byte aligned).
 * d_weight: device fp32 [k_vol][c_in][c_out], ACCUMULATED (zero it before the first
 *          call); offsets with no pair are left unchanged.
 * f16/bf16: tcgen05 per-offset gather-GEMM contracting over the pairs (MN-major operands,
 *          fp32 accumulation in TMEM, red.global.add into d_weight); c_in, c_out
 *          multiples of 16.  f32: FFMA.  Reduction order is not fixed (atomics). */
/* dst[r][0..c) += src[r][0..c) (accumulate != 0) or = src[r][0..c) (accumulate == 0, the
 * first contribution to a gradient) for r < *n_dev (or n_cap): the residual branch of a
 * backward pass (the gradient of out = conv + residual w.r.t. residual).  c % 8 == 0,
 * rows 16-byte aligned; dst and src must not overlap unless equal. */
spc_status spc_add_rows(void *dst, int64_t ld_dst, const void *src, int64_t ld_src, int64_t n_cap,
                        const int64_t *n_dev, int32_t c, int32_t dtype, int32_t accumulate, void *stream);
spc_status spc_conv_wgrad(const spc_kmap *kmap, const void *f_in, int64_t ld_in, int32_t in_dtype,
                          int32_t c_in, const void *d_out, int64_t ld_dout, int32_t c_out, float *d_weight,
                          void *stream);

/* ================================================================================
 * A13  spc_network_kmaps -- network-wide voxel indexing (§5.5)
 *
 * Phase 1: every coordinate level V_m = floor(V_0/2^m)2^m, m = 1..n_levels-1, from V_0
 * directly (Eq. (3)) in one grouped spc_downsample.  Phase 2: every map of `geoms`
 * (identical (geom, t, flags) entries are built once and shared).  No host sync:
 * level counts stay on the device.
 * level_keys_out: device buffer [n_levels][n0]; level 0 = a copy of v0_keys.
 * level_n_dev   : device int64 [n_levels].
 * maps_out_host : [n_maps] kmap structs (pointers into ws).
 * ws            : >= spc_network_workspace_size(...).
 * ================================================================================ */
size_t spc_network_workspace_size(int64_t n0, int32_t n_levels, const spc_geom *geoms_host,
                                  const int32_t *t_host, const uint32_t *flags_host, int32_t n_maps);
spc_status spc_network_kmaps(const uint64_t *v0_keys, int64_t n0, const int64_t *n0_dev,
                             spc_pack_spec spec, int32_t n_levels, const spc_geom *geoms_host,
                             const int32_t *t_host, const uint32_t *flags_host, int32_t n_maps,
                             uint64_t *level_keys_out, int64_t *level_n_dev, spc_kmap *maps_out_host,
                             uint32_t *status, void *ws, size_t ws_bytes, void *stream);

/* ================================================================================
 * Multi-GPU, one large scene: output-key ranges with input halos
 *
 * Shard r of n_shards owns the sorted outputs [out_lo, out_hi) = [r*n/R, (r+1)*n/R)
 * (n = *n_out_dev or n_out) and needs only the inputs
 *     [in_lo, in_hi) = [lb(out[out_lo] + d_min), lb(out[out_hi-1] + d_max + 1))
 * where d_min / d_max are the smallest / largest packed query offsets of the map (
 * negated for a transposed map): the keys are sorted lexicographically, so every match
 * of the shard's outputs lies in this ONE contiguous halo range.  A shard's
 * map is then spc_build_kmap(in_keys + in_lo, in_hi - in_lo, out_keys + out_lo,
 * out_hi - out_lo, ...) and its features spc_conv_forward on F_in + in_lo rows into
 * F_out + out_lo rows; the shards' maps (indices shifted back) are exactly the
 * single-device map.  Kernel maps never cross GPUs.
 * bounds_dev: device int64 [n_shards][4] = (out_lo, out_hi, in_lo, in_hi).
 * ================================================================================ */
spc_status spc_shard_ranges(const uint64_t *in_keys, int64_t n_in, const int64_t *n_in_dev, const uint64_t *out_keys,
                            int64_t n_out, const int64_t *n_out_dev, spc_pack_spec spec, spc_geom geom,
                            int32_t n_shards, int64_t *bounds_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPC_H */
