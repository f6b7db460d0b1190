// spc_host.cu -- host-side C ABI of libspc: status plumbing, pack planning, offset and
// mask helpers, and network-wide voxel indexing (A13, §5.5).
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "spc_common.cuh"

namespace spc {

static thread_local std::string g_detail;

void set_detail(const std::string &s) { g_detail = s; }

spc_status fail(spc_status st, const std::string &detail) {
    g_detail = detail;
    return st;
}

spc_status cuda_fail(cudaError_t e, const char *what) {
    g_detail = std::string(what) + ": " + cudaGetErrorString(e);
    return SPC_ERR_CUDA;
}

// process-wide tuning options (spc_set_option); performance only
static const int64_t kOptDefault[SPC_OPT_COUNT] = {0, 72, 1, 2, 1, 1, 1, 4096, 0, 1, 0, 1, 16, 0, 0, 128};
static int64_t g_opt[SPC_OPT_COUNT] = {0, 72, 1, 2, 1, 1, 1, 4096, 0, 1, 0, 1, 16, 0, 0, 128};

static unsigned long long *g_trace_buf = nullptr;
static int64_t g_trace_cap = 0;
static std::vector<std::string> g_trace_desc;

Trace trace_next(const std::string &desc) {
    Trace t{g_trace_buf, g_trace_cap, 0};
    if (g_trace_buf) {
        t.launch = (uint32_t)g_trace_desc.size();
        g_trace_desc.push_back(desc);
    }
    return t;
}

int64_t option(int o) { return (o >= 0 && o < SPC_OPT_COUNT) ? g_opt[o] : 0; }

bool pdl_enabled() { return g_opt[SPC_OPT_PDL] != 0; }

// device attributes cached per device (a process may drive several GPUs)
constexpr int MAX_DEVICES = 64;
static int g_num_sms[MAX_DEVICES];

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return (dev >= 0 && dev < MAX_DEVICES) ? dev : 0;
}

int num_sms() {
    const int dev = current_device();
    int n = g_num_sms[dev];
    if (!n) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        g_num_sms[dev] = n;
    }
    return n;
}

__global__ void k_fill_i64(int64_t *p, int64_t v) {
    pdl_wait();   // PDL launch: the predecessor has completed and flushed
    pdl_trigger(); *p = v; }
spc_status fill_i64(int64_t *p, int64_t v, cudaStream_t st) {
    SPC_CUDA(launch_pdl(k_fill_i64, dim3(1), dim3(1), 0, st, p, v));
    SPC_LAUNCH_CHECK("k_fill_i64");
    return SPC_OK;
}

}  // namespace spc

using namespace spc;

extern "C" const char *spc_status_string(int s) {
    switch (s) {
        case SPC_OK: return "SPC_OK";
        case SPC_ERR_INVALID_ARG: return "SPC_ERR_INVALID_ARG";
        case SPC_ERR_UNSUPPORTED: return "SPC_ERR_UNSUPPORTED";
        case SPC_ERR_RANGE: return "SPC_ERR_RANGE";
        case SPC_ERR_DUPLICATE: return "SPC_ERR_DUPLICATE";
        case SPC_ERR_UNSORTED: return "SPC_ERR_UNSORTED";
        case SPC_ERR_CAPACITY: return "SPC_ERR_CAPACITY";
        case SPC_ERR_WORKSPACE: return "SPC_ERR_WORKSPACE";
        case SPC_ERR_CUDA: return "SPC_ERR_CUDA";
        default: return "SPC_ERR_UNKNOWN";
    }
}

extern "C" const char *spc_last_error_detail(void) { return g_detail.c_str(); }

extern "C" int spc_version(void) { return SPC_VERSION; }

extern "C" size_t spc_kmap_struct_bytes(void) { return sizeof(spc_kmap); }

extern "C" spc_status spc_set_option(int32_t o, int64_t value) {
    if (o < 0 || o >= SPC_OPT_COUNT) return fail(SPC_ERR_INVALID_ARG, "spc_set_option: unknown option " + std::to_string(o));
    g_opt[o] = value < 0 ? kOptDefault[o] : value;
    return SPC_OK;
}

extern "C" int64_t spc_get_option(int32_t o) { return option(o); }

extern "C" spc_status spc_set_trace(void *buf, int64_t cap) {
    SPC_CHECK_ARG(cap >= 0, "cap < 0");
    g_trace_buf = static_cast<unsigned long long *>(buf);
    g_trace_cap = buf ? cap : 0;
    g_trace_desc.clear();
    return SPC_OK;
}

extern "C" const char *spc_trace_launch_desc(int32_t launch) {
    if (launch < 0 || launch >= (int32_t)g_trace_desc.size()) return "";
    return g_trace_desc[launch].c_str();
}

extern "C" spc_status spc_plan_pack(const int32_t lo[3], const int32_t hi[3], int32_t n_batch,
                                    int32_t max_out_stride, int32_t max_reach, spc_pack_spec *out) {
    SPC_CHECK_ARG(lo && hi && out, "null pointer");
    SPC_CHECK_ARG(n_batch >= 1 && max_out_stride >= 1 && max_reach >= 0, "bad n_batch/stride/reach");
    int log2s = 0;
    while ((1 << log2s) < max_out_stride) ++log2s;
    SPC_CHECK_ARG((1 << log2s) == max_out_stride, "max_out_stride must be a power of two");
    int bits[3];
    const char *axis = "xyz";
    for (int d = 0; d < 3; ++d) {
        SPC_CHECK_ARG(lo[d] <= hi[d], "lo > hi");
        const int64_t need_lo = (int64_t)lo[d] - (max_out_stride - 1) - max_reach;   // reading A4
        const int64_t need_hi = (int64_t)hi[d] + max_reach;
        int b = log2s + 1;
        while (b < 40 && (need_lo < -(1ll << (b - 1)) || need_hi > (1ll << (b - 1)) - 1)) ++b;
        bits[d] = b;
        if (b >= 40)
            return fail(SPC_ERR_RANGE, std::string("spc_plan_pack: axis ") + axis[d] + " extent does not fit");
    }
    int bb = 0;
    while ((1ll << bb) < n_batch) ++bb;
    const int total = bb + bits[0] + bits[1] + bits[2];
    if (total > 62)
        return fail(SPC_ERR_RANGE, "spc_plan_pack: needs " + std::to_string(total) + " bits (b=" +
                                       std::to_string(bb) + " x=" + std::to_string(bits[0]) + " y=" +
                                       std::to_string(bits[1]) + " z=" + std::to_string(bits[2]) + ") > 62");
    out->bits_b = bb;
    out->bits_x = bits[0];
    out->bits_y = bits[1];
    out->bits_z = bits[2];
    out->reach = max_reach;
    out->out_stride = max_out_stride;
    return SPC_OK;
}

extern "C" int64_t spc_pack_offset(spc_pack_spec s, int32_t dx, int32_t dy, int32_t dz) {
    return (int64_t)dx * (1ll << (s.bits_y + s.bits_z)) + (int64_t)dy * (1ll << s.bits_z) + (int64_t)dz;
}

extern "C" uint64_t spc_downsample_mask(spc_pack_spec s, int32_t m) {
    const int used = s.bits_b + s.bits_x + s.bits_y + s.bits_z;
    uint64_t mask = used >= 64 ? ~0ull : ((1ull << used) - 1);
    const int sh[3] = {s.bits_y + s.bits_z, s.bits_z, 0};
    for (int d = 0; d < 3; ++d)
        for (int b = 0; b < m; ++b) mask &= ~(1ull << (sh[d] + b));   // m low zeros per field
    return mask;
}

// ------------------------------------------------------------------------------------
// A13 network-wide voxel indexing
// ------------------------------------------------------------------------------------
static int log2i(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return ((1 << l) == v) ? l : -1;
}

// levels of the fine/coarse coordinate sets a map needs
static spc_status map_levels(const spc_geom &g, int n_levels, int &lev_in, int &lev_out) {
    int lf = log2i(g.tensor_stride), ls = log2i(g.stride);
    if (lf < 0 || ls < 0) return fail(SPC_ERR_INVALID_ARG, "tensor_stride and stride must be powers of two");
    int lc = lf + ls;
    if (lc >= n_levels) return fail(SPC_ERR_INVALID_ARG, "map needs a level >= n_levels");
    if (g.transposed) {
        lev_in = lc;
        lev_out = lf;
    } else {
        lev_in = lf;
        lev_out = lc;
    }
    return SPC_OK;
}

static bool same_map(const spc_geom &a, int ta, uint32_t fa, const spc_geom &b, int tb, uint32_t fb) {
    return memcmp(&a, &b, sizeof(spc_geom)) == 0 && ta == tb && fa == fb;
}

extern "C" size_t spc_network_workspace_size(int64_t n0, int32_t n_levels, const spc_geom *geoms,
                                             const int32_t *ts, const uint32_t *flags, int32_t n_maps) {
    if (n0 < 0 || n_levels < 1 || n_levels > 5) return 0;
    size_t total = align_up(spc_downsample_workspace_size(n0, n_levels > 1 ? n_levels - 1 : 1), 256);
    int64_t order_rows = 0;
    for (int i = 0; i < n_maps; ++i) {
        bool dup = false;
        for (int j = 0; j < i; ++j) dup |= same_map(geoms[i], ts[i], flags ? flags[i] : 0, geoms[j], ts[j],
                                                    flags ? flags[j] : 0);
        if (dup) continue;
        total += align_up(kmap_bytes_batched(geoms[i], ts[i], flags ? flags[i] : 0, n0), 256);
        order_rows += (int64_t)kmap_order_rows(geoms[i], ts[i], flags ? flags[i] : 0, n0);
    }
    // one density-order sort over all ordered maps (end of the workspace)
    total += align_up(kmap_order_scratch_bytes(order_rows), 256);
    return total + 256;
}

extern "C" spc_status spc_network_kmaps(const uint64_t *v0_keys, int64_t n0, const int64_t *n0_dev,
                                        spc_pack_spec spec, int32_t n_levels, const spc_geom *geoms,
                                        const int32_t *ts, const uint32_t *flags, int32_t n_maps,
                                        uint64_t *level_keys, int64_t *level_n_dev, spc_kmap *maps_out,
                                        uint32_t *status, void *ws, size_t ws_bytes, void *stream) {
    SPC_CHECK_ARG(n0 >= 0 && n_levels >= 1 && n_levels <= 5 && n_maps >= 0, "bad sizes");
    SPC_CHECK_ARG(level_keys && level_n_dev && (n_maps == 0 || (geoms && ts && maps_out)), "null pointer");
    if (ws_bytes < spc_network_workspace_size(n0, n_levels, geoms, ts, flags, n_maps))
        return fail(SPC_ERR_WORKSPACE, "spc_network_kmaps: ws too small");
    cudaStream_t st = as_stream(stream);
    char *base = static_cast<char *>(ws);
    const size_t ds_bytes = spc_downsample_workspace_size(n0, n_levels > 1 ? n_levels - 1 : 1);
    size_t off = align_up(ds_bytes, 256);

    // ---- phase 1: level 0 = V_0, levels 1.. = floor(V_0 / 2^m) 2^m (Eq. 3) -----------
    if (n0 > 0) SPC_CUDA(cudaMemcpyAsync(level_keys, v0_keys, sizeof(uint64_t) * n0, cudaMemcpyDeviceToDevice, st));
    if (n0_dev) SPC_CUDA(cudaMemcpyAsync(level_n_dev, n0_dev, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    else {
        spc_status s = fill_i64(level_n_dev, n0, st);
        if (s != SPC_OK) return s;
    }
    if (n_levels > 1) {
        int32_t m[4];
        for (int l = 1; l < n_levels; ++l) m[l - 1] = l;
        spc_status s = spc_downsample(v0_keys, n0, n0_dev, spec, n_levels - 1, m, level_keys + n0, level_n_dev + 1,
                                      base, ds_bytes, stream);
        if (s != SPC_OK) return s;
    }
    // ---- phase 2: every distinct map, one grouped launch ---------------------------------
    int64_t order_rows = 0;
    size_t maps_bytes = 0;
    for (int i = 0; i < n_maps; ++i) {
        const uint32_t fi = flags ? flags[i] : 0;
        bool dup = false;
        for (int j = 0; j < i; ++j) dup |= same_map(geoms[i], ts[i], fi, geoms[j], ts[j], flags ? flags[j] : 0);
        if (dup) continue;
        maps_bytes += align_up(kmap_bytes_batched(geoms[i], ts[i], fi, n0), 256);
        order_rows += (int64_t)kmap_order_rows(geoms[i], ts[i], fi, n0);
    }
    kmap_defer_begin(base + off + maps_bytes, kmap_order_scratch_bytes(order_rows), order_rows);
    for (int i = 0; i < n_maps; ++i) {
        const uint32_t fi = flags ? flags[i] : 0;
        int dup = -1;
        for (int j = 0; j < i && dup < 0; ++j)
            if (same_map(geoms[i], ts[i], fi, geoms[j], ts[j], flags ? flags[j] : 0)) dup = j;
        if (dup >= 0) {
            maps_out[i] = maps_out[dup];
            continue;
        }
        int li, lo;
        spc_status s = map_levels(geoms[i], n_levels, li, lo);
        if (s != SPC_OK) {
            kmap_defer_abort();
            return s;
        }
        const size_t bytes = kmap_bytes_batched(geoms[i], ts[i], fi, n0);
        s = spc_build_kmap(level_keys + (size_t)li * n0, n0, level_n_dev + li, level_keys + (size_t)lo * n0, n0,
                           level_n_dev + lo, spec, geoms[i], ts[i], fi, base + off, bytes, status, &maps_out[i],
                           stream);
        if (s != SPC_OK) {
            kmap_defer_abort();   // leaves no half-open batch behind
            return s;
        }
        off += align_up(bytes, 256);
    }
    return kmap_defer_end(st);
}
