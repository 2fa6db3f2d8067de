// matq_glue.cu -- the bf16 glue of the full-model decode harness (SURVEY 8(f)
// rank 3, llama.py) fused into three row kernels, so that a Llama block's
// step is 4 sliced linears + 3 glue launches + attention instead of ~30 small
// torch kernels.  Not part of the sliced-linear deliverable: plain CUDA-core
// code: one CTA per token row (SiLU: a row split over CTAs), 16-byte accesses,
// programmatic dependent launch.
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

__device__ __forceinline__ void glue_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void glue_pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// One CTA per row; each thread owns 8 consecutive elements (one 16-byte load of x and of
// delta) -- h <= 8 * 1024 -- so the row is read once and kept in registers.
__global__ void k_add_rmsnorm(__nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ delta,
                              const float* __restrict__ w, __nv_bfloat16* __restrict__ y, int h, float eps) {
    __shared__ float red[32];
    glue_pdl_wait();  // x / delta come from the previous kernel
    glue_pdl_launch();
    const int b = blockIdx.x;
    const int i0 = threadIdx.x * 8;
    const bool act = i0 < h;
    __nv_bfloat16* xr = x + (long long)b * h;
    float v[8];
    float ss = 0.0f;
    if (act) {
        const uint4 xv = *reinterpret_cast<const uint4*>(xr + i0);
        const __nv_bfloat16* xe = reinterpret_cast<const __nv_bfloat16*>(&xv);
        if (delta) {
            const uint4 dv = *reinterpret_cast<const uint4*>(delta + (long long)b * h + i0);
            const __nv_bfloat16* de = reinterpret_cast<const __nv_bfloat16*>(&dv);
            uint4 ov;
            __nv_bfloat16* oe = reinterpret_cast<__nv_bfloat16*>(&ov);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                oe[j] = __float2bfloat16_rn(bf(xe[j]) + bf(de[j]));  // the residual stream is bf16
                v[j] = bf(oe[j]);
            }
            *reinterpret_cast<uint4*>(xr + i0) = ov;
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = bf(xe[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) ss += v[j] * v[j];
    }
    const float inv = rsqrtf(block_sum(ss, red) / (float)h + eps);
    if (act) {
        uint4 ov;
        __nv_bfloat16* oe = reinterpret_cast<__nv_bfloat16*>(&ov);
        const float4 w0 = *reinterpret_cast<const float4*>(w + i0), w1 = *reinterpret_cast<const float4*>(w + i0 + 4);
        const float ww[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) oe[j] = __float2bfloat16_rn(v[j] * inv * ww[j]);
        *reinterpret_cast<uint4*>(y + (long long)b * h + i0) = ov;
    }
}

// qkv row: [q: nh*hd | k: nkv*hd | v: nkv*hd]; caches (B, nkv, T, hd).  One warp per
// q / k head (hd a multiple of 64, <= 256): optional per-head RMSNorm (Qwen3's q_norm /
// k_norm: qn / kn non-null; fp32 math, rounded to bf16 like torch), then the rotary
// rotation, rounded to bf16 per torch op.
__global__ void k_rope_kv(const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ cosv,
                          const __nv_bfloat16* __restrict__ sinv, __nv_bfloat16* __restrict__ q,
                          __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, int nh, int nkv, int hd,
                          int T, int pos, const float* __restrict__ qn, const float* __restrict__ kn, float eps) {
    glue_pdl_wait();
    glue_pdl_launch();
    const int b = blockIdx.x, half = hd >> 1, per = half >> 5;  // elements per lane in each half (<= 4)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const __nv_bfloat16* row = qkv + (long long)b * (nh + 2 * nkv) * hd;
    for (int head = warp; head < nh + nkv; head += nw) {
        const __nv_bfloat16* src = row + head * hd;
        const float* nw_ = head < nh ? qn : kn;
        float x1[4], x2[4];
        float ss = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i < per) {
                x1[i] = bf(src[lane + 32 * i]);
                x2[i] = bf(src[half + lane + 32 * i]);
                ss += x1[i] * x1[i] + x2[i] * x2[i];
            }
        }
        if (nw_) {
#pragma unroll
            for (int sh = 16; sh >= 1; sh >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, sh);
            const float inv = rsqrtf(ss / (float)hd + eps);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (i < per) {
                    x1[i] = bf(__float2bfloat16_rn(x1[i] * inv * nw_[lane + 32 * i]));
                    x2[i] = bf(__float2bfloat16_rn(x2[i] * inv * nw_[half + lane + 32 * i]));
                }
            }
        }
        __nv_bfloat16* dst = head < nh ? q + ((long long)b * nh + head) * hd
                                       : kc + (((long long)b * nkv + (head - nh)) * T + pos) * hd;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i < per) {
                const int j = lane + 32 * i;
                const float c = bf(cosv[j]), s = bf(sinv[j]);
                const float o1 = bf(__float2bfloat16_rn(bf(__float2bfloat16_rn(x1[i] * c)) - bf(__float2bfloat16_rn(x2[i] * s))));
                const float o2 = bf(__float2bfloat16_rn(bf(__float2bfloat16_rn(x2[i] * c)) + bf(__float2bfloat16_rn(x1[i] * s))));
                dst[j] = __float2bfloat16_rn(o1);
                dst[j + half] = __float2bfloat16_rn(o2);
            }
        }
    }
    for (int i = threadIdx.x; i < nkv * hd; i += blockDim.x) {
        const int head = i / hd, j = i - head * hd;
        vc[(((long long)b * nkv + head) * T + pos) * hd + j] = row[(nh + nkv) * hd + i];
    }
}

// grid (rows, ceil(inter / (8 * 256))): 8 consecutive columns per thread (16-byte loads)
__global__ void k_silu_mul(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ y, int inter) {
    glue_pdl_wait();
    glue_pdl_launch();
    const int b = blockIdx.x;
    const int i0 = (blockIdx.y * blockDim.x + threadIdx.x) * 8;
    if (i0 >= inter) return;
    const __nv_bfloat16* g = gu + (long long)b * 2 * inter;
    const uint4 gv = *reinterpret_cast<const uint4*>(g + i0), uv = *reinterpret_cast<const uint4*>(g + inter + i0);
    const __nv_bfloat16* ge = reinterpret_cast<const __nv_bfloat16*>(&gv);
    const __nv_bfloat16* ue = reinterpret_cast<const __nv_bfloat16*>(&uv);
    uint4 ov;
    __nv_bfloat16* oe = reinterpret_cast<__nv_bfloat16*>(&ov);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float gf = bf(ge[j]);
        const float sv = bf(__float2bfloat16_rn(gf / (1.0f + __expf(-gf))));  // torch: silu in bf16
        oe[j] = __float2bfloat16_rn(sv * bf(ue[j]));
    }
    *reinterpret_cast<uint4*>(y + (long long)b * inter + i0) = ov;
}

}  // namespace

// programmatic dependent launch: the kernel's prologue overlaps the previous
// kernel's tail; it waits (griddepcontrol.wait) before touching its inputs
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

cudaError_t launch_add_rmsnorm(void* x, const void* delta, const float* w, void* y, int B, int h, float eps,
                               cudaStream_t s) {
    if (h % 8 || h > 8 * 1024) return cudaErrorInvalidValue;
    const int threads = ((h / 8 + 31) / 32) * 32;
    return launch_pdl(k_add_rmsnorm, dim3(B), dim3(threads), s, reinterpret_cast<__nv_bfloat16*>(x),
                      reinterpret_cast<const __nv_bfloat16*>(delta), w, reinterpret_cast<__nv_bfloat16*>(y), h,
                      eps);
}

cudaError_t launch_rope_kv(const void* qkv, const void* cosv, const void* sinv, void* q, void* kc, void* vc, int B,
                           int nh, int nkv, int hd, int T, int pos, const float* qn, const float* kn, float eps,
                           cudaStream_t s) {
    if (hd % 64 || hd > 256) return cudaErrorInvalidValue;
    return launch_pdl(k_rope_kv, dim3(B), dim3(512), s, reinterpret_cast<const __nv_bfloat16*>(qkv),
                      reinterpret_cast<const __nv_bfloat16*>(cosv), reinterpret_cast<const __nv_bfloat16*>(sinv),
                      reinterpret_cast<__nv_bfloat16*>(q), reinterpret_cast<__nv_bfloat16*>(kc),
                      reinterpret_cast<__nv_bfloat16*>(vc), nh, nkv, hd, T, pos, qn, kn, eps);
}

cudaError_t launch_silu_mul(const void* gu, void* y, int B, int inter, cudaStream_t s) {
    if (inter % 8) return cudaErrorInvalidValue;
    return launch_pdl(k_silu_mul, dim3(B, (inter / 8 + 255) / 256), dim3(256), s,
                      reinterpret_cast<const __nv_bfloat16*>(gu), reinterpret_cast<__nv_bfloat16*>(y), inter);
}

}  // namespace mq
