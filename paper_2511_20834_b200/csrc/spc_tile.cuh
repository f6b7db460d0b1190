// spc_tile.cuh -- epilogue helpers shared by the tcgen05 feature kernels (internal).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "spc.h"

namespace spc {

enum OutKind : int { OUT_FINAL = 0, OUT_F32_STORE = 1, OUT_F32_RED = 2 };

// fused epilogue of a final store (spc_epilogue): y = acc * scale[c] +
// shift[c] (inference batch norm, folded), then + residual, then max(y, 0) if relu
struct Epi {
    const float *scale;   // nullable
    const float *shift;   // nullable
    int relu;
};
__host__ __device__ __forceinline__ bool epi_on(const Epi &e) { return e.scale || e.shift || e.relu; }
// n consecutive columns starting at col: the affine part (before the residual)
template <int N>
__device__ __forceinline__ void epi_affine(const Epi &e, float (&f)[N], int col) {
    if (e.scale) {
#pragma unroll
        for (int i = 0; i < N; ++i) f[i] *= __ldg(e.scale + col + i);
    }
    if (e.shift) {
#pragma unroll
        for (int i = 0; i < N; ++i) f[i] += __ldg(e.shift + col + i);
    }
}
template <int N>
__device__ __forceinline__ void epi_relu(const Epi &e, float (&f)[N]) {
    if (e.relu) {
#pragma unroll
        for (int i = 0; i < N; ++i) f[i] = fmaxf(f[i], 0.f);
    }
}

__device__ __forceinline__ float to_f(uint32_t u) { return __uint_as_float(u); }

__device__ __forceinline__ uint32_t pack2(float a, float b, int dt) {
    if (dt == SPC_BF16) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ float2 unpack2(uint32_t u, int dt) {
    if (dt == SPC_BF16) return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162 *>(&u));
    return __half22float2(*reinterpret_cast<__half2 *>(&u));
}

// the affine part of the epilogue applied in place to n (16 or 32) accumulator values of
// columns col.. (callers run it before store_row, which adds the residual and the ReLU)
__device__ __forceinline__ void epi_affine_u32(const Epi &e, uint32_t (&v)[32], int col, int n) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if (q * 4 < n) {
            const float4 s = e.scale ? __ldg(reinterpret_cast<const float4 *>(e.scale + col) + q) : make_float4(1.f, 1.f, 1.f, 1.f);
            const float4 b = e.shift ? __ldg(reinterpret_cast<const float4 *>(e.shift + col) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            v[4 * q] = __float_as_uint(fmaf(to_f(v[4 * q]), s.x, b.x));
            v[4 * q + 1] = __float_as_uint(fmaf(to_f(v[4 * q + 1]), s.y, b.y));
            v[4 * q + 2] = __float_as_uint(fmaf(to_f(v[4 * q + 2]), s.z, b.z));
            v[4 * q + 3] = __float_as_uint(fmaf(to_f(v[4 * q + 3]), s.w, b.w));
        }
}

// store 'n' (16 or 32) fp32 values of one row to the output (fully unrolled: registers only);
// OUT_FINAL: + residual, then the epilogue's ReLU (its affine part was applied by the caller)
template <bool EPI = true, class P>
__device__ __forceinline__ void store_row(const P &p, int64_t row, int col, const uint32_t (&v)[32], int n) {
    const bool epi = EPI && p.out_kind == OUT_FINAL && p.epi.relu;
    if (p.out_kind == OUT_FINAL && p.out_dtype != SPC_F32) {
        const uint4 *rp = p.residual
                              ? reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(p.residual) + row * p.ld_res + col)
                              : nullptr;
        uint4 *op = reinterpret_cast<uint4 *>(static_cast<uint16_t *>(p.out) + row * p.ld_out + col);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (q * 8 < n) {
                float f[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = to_f(v[q * 8 + e]);
                if (rp) {
                    const uint4 u = rp[q];
                    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 r2 = unpack2(w[e], p.out_dtype);
                        f[2 * e] += r2.x;
                        f[2 * e + 1] += r2.y;
                    }
                }
                if (epi) epi_relu(p.epi, f);
                op[q] = make_uint4(pack2(f[0], f[1], p.out_dtype), pack2(f[2], f[3], p.out_dtype),
                                   pack2(f[4], f[5], p.out_dtype), pack2(f[6], f[7], p.out_dtype));
            }
        }
    } else {
        float *op = static_cast<float *>(p.out) + row * p.ld_out + col;
        const float *rp = (p.out_kind == OUT_FINAL && p.residual)
                              ? static_cast<const float *>(p.residual) + row * p.ld_res + col
                              : nullptr;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q * 4 < n) {
                float f[4] = {to_f(v[4 * q]), to_f(v[4 * q + 1]), to_f(v[4 * q + 2]), to_f(v[4 * q + 3])};
                if (rp) {
                    const float4 r = reinterpret_cast<const float4 *>(rp)[q];
                    f[0] += r.x; f[1] += r.y; f[2] += r.z; f[3] += r.w;
                }
                if (epi) epi_relu(p.epi, f);
                reinterpret_cast<float4 *>(op)[q] = make_float4(f[0], f[1], f[2], f[3]);
            }
        }
    }
}

}  // namespace spc
