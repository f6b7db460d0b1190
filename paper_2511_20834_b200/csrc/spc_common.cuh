// spc_common.cuh -- internal helpers of libspc (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "spc.h"

namespace spc {

// ------------------------------------------------------------------------------------
// host-side error plumbing
// ------------------------------------------------------------------------------------
void set_detail(const std::string &s);
spc_status fail(spc_status st, const std::string &detail);
spc_status cuda_fail(cudaError_t e, const char *what);

#define SPC_CHECK_ARG(cond, msg)                                                         \
    do {                                                                                 \
        if (!(cond)) return ::spc::fail(SPC_ERR_INVALID_ARG, std::string(__func__) + ": " + (msg)); \
    } while (0)

#define SPC_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t _e = (call);                                                         \
        if (_e != cudaSuccess) return ::spc::cuda_fail(_e, #call);                       \
    } while (0)

#define SPC_LAUNCH_CHECK(name)                                                           \
    do {                                                                                 \
        cudaError_t _e = cudaGetLastError();                                             \
        if (_e != cudaSuccess) return ::spc::cuda_fail(_e, name);                        \
    } while (0)

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// simple bump allocator over a caller workspace
struct Bump {
    char *base;
    size_t cap, used;
    Bump(void *b, size_t c) : base(static_cast<char *>(b)), cap(c), used(0) {}
    template <class T>
    T *take(size_t count) {
        used = align_up(used, 256);
        T *p = reinterpret_cast<T *>(base + used);
        used += count * sizeof(T);
        return p;
    }
    bool ok() const { return used <= cap; }
};
// size-only twin of Bump
struct Sizer {
    size_t used = 0;
    template <class T>
    void take(size_t count) {
        used = align_up(used, 256);
        used += count * sizeof(T);
    }
};

int num_sms();           // SM count of the current device (cached per device)
int current_device();
bool pdl_enabled();      // programmatic dependent launch (spc_set_option(SPC_OPT_PDL, 0) turns it off)
int64_t option(int o);   // spc_set_option value

// Launch with programmatic stream serialisation (PDL): the kernel may start while the
// previous kernel in the stream drains.  Every kernel launched this way executes
// pdl_wait() before touching memory another kernel writes, and pdl_trigger() only after
// that wait, so when a kernel starts its predecessor's predecessor has completed.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// the same with a thread-block cluster of `cluster_x` CTAs (CTA pairs, cta_group::2)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               int cluster_x, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster_x;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------------------------
// device helpers
// ------------------------------------------------------------------------------------
// PDL: wait for the preceding kernel's completion (and memory flush); no-op when the
// kernel was launched without the attribute
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// PDL: let the next kernel in the stream begin its prologue
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// device-side event trace (spc_set_trace): null buffer = off
struct Trace {
    unsigned long long *buf;
    int64_t cap;
    uint32_t launch;
};
static __device__ __noinline__ void trace_record(const Trace &t, int ev, uint32_t aux);
// launch-level events (entry, PDL release, setup, exit): a predicated out-of-line call
__device__ __forceinline__ void trace_event(const Trace &t, int ev, uint32_t aux) {
    if (t.buf) trace_record(t, ev, aux);
}
// per-tile events (records, first full stage, commits, epilogues) sit in the pipeline
// loops, where even a predicated call measurably costs (~1% of a C2 step): they are
// compiled only into the tracing build of the library
// (python -m paper_2511_20834_b200.build --exp trace -DSPC_TRACE_TILES; scripts/timeline.py)
__device__ __forceinline__ void trace_tile_event(const Trace &t, int ev, uint32_t aux) {
#ifdef SPC_TRACE_TILES
    if (t.buf) trace_record(t, ev, aux);
#else
    (void)t; (void)ev; (void)aux;
#endif
}
static __device__ __noinline__ void trace_record(const Trace &t, int ev, uint32_t aux) {
    unsigned long long ts;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
    const unsigned long long i = atomicAdd(t.buf, 1ull);
    if ((int64_t)i < t.cap) {
        t.buf[1 + 2 * i] = ts;
        t.buf[2 + 2 * i] = ((unsigned long long)t.launch << 48) | ((unsigned long long)ev << 40) |
                           ((unsigned long long)(blockIdx.x & 0xffff) << 24) | (aux & 0xffffffu);
    }
}
// host: the trace descriptor for the next launch (launch numbered, described for the log)
Trace trace_next(const std::string &desc);

__device__ __forceinline__ int64_t dev_count(int64_t cap, const int64_t *n_dev) {
    if (!n_dev) return cap;
    int64_t n = *n_dev;
    return n < cap ? n : cap;
}

__device__ __forceinline__ unsigned lane_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
    return r;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

}  // namespace spc

// internal entry points shared between translation units
namespace spc {
// radix sort of (keys, optional int32 values) over bits [0, n_bits); result in keys_out / vals_out
size_t radix_sort_workspace(int64_t n, bool with_vals);
spc_status radix_sort(const uint32_t *keys_in, const int32_t *vals_in, int64_t n, const int64_t *n_dev, int n_bits,
                      uint32_t *keys_out, int32_t *vals_out, void *ws, size_t ws_bytes, cudaStream_t st, bool hist_done);
spc_status flag_unsorted(const void *keys, int key_bytes, int64_t n_cap, const int64_t *n_dev, uint32_t *status,
                         cudaStream_t st);
spc_status radix_sort(const uint64_t *keys_in, const int32_t *vals_in /*nullable: identity*/, int64_t n,
                      const int64_t *n_dev, int n_bits, uint64_t *keys_out, int32_t *vals_out /*nullable*/,
                      void *ws, size_t ws_bytes, cudaStream_t st, bool hist_done);
}  // namespace spc

namespace spc {
// network-wide phase 2: spc_build_kmap calls between begin/end are collected and built by
// one grouped launch (spc_kmap.cu)
void kmap_defer_begin(void *order_scratch, size_t order_scratch_bytes, int64_t order_rows);
size_t kmap_bytes_batched(spc_geom geom, int32_t t, uint32_t flags, int64_t n_out);   // map buffer in a batch
size_t kmap_order_rows(spc_geom geom, int32_t t, uint32_t flags, int64_t n_out);      // rows it adds to the order sort
size_t kmap_order_scratch_bytes(int64_t rows);
void kmap_defer_abort();
spc_status kmap_defer_end(cudaStream_t st);
}  // namespace spc
