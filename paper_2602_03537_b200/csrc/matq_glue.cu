// matq_glue.cu -- the bf16 glue of the full-model decode harness (SURVEY 8(f)
// rank 3, llama.py) fused into three row kernels, so that a Llama block's
// step is 4 sliced linears + 3 glue launches + attention instead of ~30 small
// torch kernels.  Not part of the sliced-linear deliverable: plain CUDA-core
// code, one CTA per token row.
//   * k_add_rmsnorm: x += delta (the residual), y = x * rsqrt(mean(x^2) + eps) * w
//   * k_rope_kv:     rotary embedding (rotate-half form) of q and k from the fused
//                    qkv row, q -> (B, nh, hd), k and v written into the caches at
//                    position pos
//   * k_silu_mul:    y = silu(g) * u for gu = [g | u]
// Arithmetic in fp32, bf16 in and out (the torch reference rounds the same
// intermediates; tests compare within bf16 tolerance).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "matq_internal.h"

namespace mq {
namespace {

__device__ __forceinline__ float bf(const __nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    v = lane < nw ? red[lane] : 0.0f;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    __syncthreads();
    return v;
}

__global__ void k_add_rmsnorm(__nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ delta,
                              const float* __restrict__ w, __nv_bfloat16* __restrict__ y, int h, float eps) {
    __shared__ float red[32];
    const int b = blockIdx.x;
    __nv_bfloat16* xr = x + (long long)b * h;
    const __nv_bfloat16* dr = delta ? delta + (long long)b * h : nullptr;
    __nv_bfloat16* yr = y + (long long)b * h;
    float ss = 0.0f;
    for (int i = threadIdx.x; i < h; i += blockDim.x) {
        float v = bf(xr[i]);
        if (dr) {
            v = bf(__float2bfloat16_rn(v + bf(dr[i])));  // the residual stream is bf16
            xr[i] = __float2bfloat16_rn(v);
        }
        ss += v * v;
    }
    const float inv = rsqrtf(block_sum(ss, red) / (float)h + eps);
    for (int i = threadIdx.x; i < h; i += blockDim.x) yr[i] = __float2bfloat16_rn(bf(xr[i]) * inv * w[i]);
}

// qkv row: [q: nh*hd | k: nkv*hd | v: nkv*hd]; caches (B, nkv, T, hd)
__global__ void k_rope_kv(const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ cosv,
                          const __nv_bfloat16* __restrict__ sinv, __nv_bfloat16* __restrict__ q,
                          __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, int nh, int nkv, int hd,
                          int T, int pos) {
    const int b = blockIdx.x, half = hd >> 1;
    const __nv_bfloat16* row = qkv + (long long)b * (nh + 2 * nkv) * hd;
    // q and k heads: (x1, x2) -> (x1 c - x2 s, x2 c + x1 s), rounded to bf16 like torch
    for (int i = threadIdx.x; i < (nh + nkv) * half; i += blockDim.x) {
        const int head = i / half, j = i - head * half;
        const __nv_bfloat16* src = row + head * hd;
        const float x1 = bf(src[j]), x2 = bf(src[j + half]);
        const float c = bf(cosv[j]), s = bf(sinv[j]);
        const float o1 = bf(__float2bfloat16_rn(bf(__float2bfloat16_rn(x1 * c)) - bf(__float2bfloat16_rn(x2 * s))));
        const float o2 = bf(__float2bfloat16_rn(bf(__float2bfloat16_rn(x2 * c)) + bf(__float2bfloat16_rn(x1 * s))));
        __nv_bfloat16* dst;
        if (head < nh) {
            dst = q + ((long long)b * nh + head) * hd;
        } else {
            dst = kc + (((long long)b * nkv + (head - nh)) * T + pos) * hd;
        }
        dst[j] = __float2bfloat16_rn(o1);
        dst[j + half] = __float2bfloat16_rn(o2);
    }
    for (int i = threadIdx.x; i < nkv * hd; i += blockDim.x) {
        const int head = i / hd, j = i - head * hd;
        vc[(((long long)b * nkv + head) * T + pos) * hd + j] = row[(nh + nkv) * hd + i];
    }
}

__global__ void k_silu_mul(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ y, int inter) {
    const int b = blockIdx.x;
    const __nv_bfloat16* g = gu + (long long)b * 2 * inter;
    for (int i = threadIdx.x; i < inter; i += blockDim.x) {
        const float gv = bf(g[i]);
        const float sv = bf(__float2bfloat16_rn(gv / (1.0f + __expf(-gv))));  // torch: silu in bf16
        y[(long long)b * inter + i] = __float2bfloat16_rn(sv * bf(g[inter + i]));
    }
}

}  // namespace

cudaError_t launch_add_rmsnorm(void* x, const void* delta, const float* w, void* y, int B, int h, float eps,
                               cudaStream_t s) {
    k_add_rmsnorm<<<B, 512, 0, s>>>(reinterpret_cast<__nv_bfloat16*>(x),
                                    reinterpret_cast<const __nv_bfloat16*>(delta), w,
                                    reinterpret_cast<__nv_bfloat16*>(y), h, eps);
    return cudaGetLastError();
}

cudaError_t launch_rope_kv(const void* qkv, const void* cosv, const void* sinv, void* q, void* kc, void* vc, int B,
                           int nh, int nkv, int hd, int T, int pos, cudaStream_t s) {
    k_rope_kv<<<B, 256, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(qkv),
                                reinterpret_cast<const __nv_bfloat16*>(cosv),
                                reinterpret_cast<const __nv_bfloat16*>(sinv), reinterpret_cast<__nv_bfloat16*>(q),
                                reinterpret_cast<__nv_bfloat16*>(kc), reinterpret_cast<__nv_bfloat16*>(vc), nh, nkv,
                                hd, T, pos);
    return cudaGetLastError();
}

cudaError_t launch_silu_mul(const void* gu, void* y, int B, int inter, cudaStream_t s) {
    k_silu_mul<<<B, 512, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(gu), reinterpret_cast<__nv_bfloat16*>(y),
                                 inter);
    return cudaGetLastError();
}

}  // namespace mq
