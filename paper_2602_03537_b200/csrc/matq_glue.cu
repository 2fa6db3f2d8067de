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

// Single-query decode attention with the rotary step fused in: one CTA per (q head,
// batch row), 256 threads.  The q head and its kv head's new k are RMS-normed (Qwen3,
// optional) and rotated exactly as k_rope_kv does (bf16 per op); the first q head of each
// kv head writes the new k / v into the caches at pos; every CTA scores its q against
// cache rows [0, pos) plus the new k (kept in shared memory: no cross-CTA ordering), with an
// fp32 softmax (scale 1/sqrt(hd)) and an fp32 weighted sum of V -> bf16 att row.  The work
// of torch SDPA (GQA) + k_rope_kv in one launch per layer.  Latency-shaped: every global
// load of the first 256 keys (K row of key tid; V of keys ks + i KS, i < 16, for the
// thread's 8-dim group) is issued at entry together with the q / k / v rows, so the kernel
// waits on memory about once; longer contexts loop over the rest.
constexpr int kAttnThreads = 256;

template <int HD>
__global__ void __launch_bounds__(kAttnThreads)
k_attn_decode(const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ cosv,
              const __nv_bfloat16* __restrict__ sinv, const float* __restrict__ qn, const float* __restrict__ kn,
              float eps, __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
              const int* __restrict__ kv_of_q, __nv_bfloat16* __restrict__ att, int nh, int nkv, int T, int pos) {
    constexpr int HALF = HD / 2, DG = HD / 8, KS = kAttnThreads / DG, VPF = kAttnThreads / KS;  // VPF = DG
    __shared__ __align__(16) float qs[HD];
    __shared__ float kns[HD], vns[HD];
    __shared__ float red[32];
    __shared__ __align__(16) float part[KS][HD + 4];
    extern __shared__ float sc[];  // pos + 1 scores
    glue_pdl_wait();
    glue_pdl_launch();
    const int h = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
    const int j = kv_of_q[h];
    const __nv_bfloat16* row = qkv + (long long)b * (nh + 2 * nkv) * HD;
    const __nv_bfloat16* kr = kc + ((long long)b * nkv + j) * T * HD;
    const __nv_bfloat16* vr = vc + ((long long)b * nkv + j) * T * HD;
    const int dg = tid % DG, ks = tid / DG;
    const uint4* vp = reinterpret_cast<const uint4*>(vr) + dg;
    // ---- every load the first pass needs, issued up front ----
    const int jj = tid < HALF ? tid : tid - HALF;
    float qx = 0.f, kx = 0.f, vx = 0.f, cs = 0.f, sn = 0.f, qw = 0.f, kw = 0.f;
    if (tid < HD) {
        qx = bf(row[h * HD + tid]);
        kx = bf(row[(nh + j) * HD + tid]);
        vx = bf(row[(nh + nkv + j) * HD + tid]);
        cs = bf(cosv[jj]);
        sn = bf(sinv[jj]);
        if (qn) {
            qw = qn[tid];
            kw = kn[tid];
        }
    }
    // K: coalesced -- a key row is read by DG consecutive lanes (16 bytes each); a warp covers
    // KPW keys per round, the CTA KPR; the first NR rounds (256 keys) are prefetched
    constexpr int KPW = 32 / DG, KPR = (kAttnThreads / 32) * KPW, NR = 256 / KPR;
    const int warp = tid >> 5, lane = tid & 31, dch = lane % DG, ksub = lane / DG;
    const uint4* kbase = reinterpret_cast<const uint4*>(kr) + dch;
    auto key_of = [&](int k) { return k * KPR + warp * KPW + ksub; };
    uint4 kreg[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        const int t = key_of(k);
        kreg[k] = t < pos ? __ldg(kbase + (long long)t * DG) : make_uint4(0u, 0u, 0u, 0u);
    }
    uint4 vreg[VPF];
#pragma unroll
    for (int i = 0; i < VPF; ++i) {
        const int t = ks + i * KS;
        vreg[i] = t < pos ? __ldg(vp + (long long)t * DG) : make_uint4(0u, 0u, 0u, 0u);
    }
    // ---- q head h and k head j: optional RMSNorm, then rotate (k_rope_kv's arithmetic) ----
    if (qn) {
        const float iq = rsqrtf(block_sum(qx * qx, red) / (float)HD + eps);
        const float ik = rsqrtf(block_sum(kx * kx, red) / (float)HD + eps);
        qx = bf(__float2bfloat16_rn(qx * iq * qw));
        kx = bf(__float2bfloat16_rn(kx * ik * kw));
    }
    if (tid < HD) {
        qs[tid] = qx;
        kns[tid] = kx;
        vns[tid] = vx;
    }
    __syncthreads();
    float qo = 0.f, ko = 0.f;
    if (tid < HD) {
        const float q1 = qs[jj], q2 = qs[jj + HALF], k1 = kns[jj], k2 = kns[jj + HALF];
        if (tid < HALF) {
            qo = bf(__float2bfloat16_rn(bf(__float2bfloat16_rn(q1 * cs)) - bf(__float2bfloat16_rn(q2 * sn))));
            ko = bf(__float2bfloat16_rn(bf(__float2bfloat16_rn(k1 * cs)) - bf(__float2bfloat16_rn(k2 * sn))));
        } else {
            qo = bf(__float2bfloat16_rn(bf(__float2bfloat16_rn(q2 * cs)) + bf(__float2bfloat16_rn(q1 * sn))));
            ko = bf(__float2bfloat16_rn(bf(__float2bfloat16_rn(k2 * cs)) + bf(__float2bfloat16_rn(k1 * sn))));
        }
    }
    __syncthreads();
    if (tid < HD) {
        qs[tid] = qo;
        kns[tid] = ko;
        // the first q head of kv head j publishes the new k / v into the caches
        if (h == 0 || kv_of_q[h - 1] != j) {
            kc[(((long long)b * nkv + j) * T + pos) * HD + tid] = __float2bfloat16_rn(ko);
            vc[(((long long)b * nkv + j) * T + pos) * HD + tid] = __float2bfloat16_rn(vx);
        }
    }
    __syncthreads();
    // ---- scores: thread t owns keys t, t + 256, ...; the new key (index pos) from shared memory ----
    const float scale = rsqrtf((float)HD);
    const float4 qa = *reinterpret_cast<const float4*>(qs + 8 * dch);
    const float4 qb = *reinterpret_cast<const float4*>(qs + 8 * dch + 4);
    auto dot8 = [&](const uint4& u) {  // this lane's 8 dims; summed over the key's DG lanes
        const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&u);
        float d = 0.0f;
        float2 f;
        f = __bfloat1622float2(e[0]); d = fmaf(qa.x, f.x, d); d = fmaf(qa.y, f.y, d);
        f = __bfloat1622float2(e[1]); d = fmaf(qa.z, f.x, d); d = fmaf(qa.w, f.y, d);
        f = __bfloat1622float2(e[2]); d = fmaf(qb.x, f.x, d); d = fmaf(qb.y, f.y, d);
        f = __bfloat1622float2(e[3]); d = fmaf(qb.z, f.x, d); d = fmaf(qb.w, f.y, d);
#pragma unroll
        for (int o = DG / 2; o >= 1; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        return d;
    };
    float mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        const float d = dot8(kreg[k]) * scale;
        const int t = key_of(k);
        if (dch == 0 && t < pos) {
            sc[t] = d;
            mx = fmaxf(mx, d);
        }
    }
    for (int k = NR; k * KPR < pos; ++k) {  // contexts past 256 keys
        const int t = key_of(k);
        const uint4 u = t < pos ? __ldg(kbase + (long long)t * DG) : make_uint4(0u, 0u, 0u, 0u);
        const float d = dot8(u) * scale;
        if (dch == 0 && t < pos) {
            sc[t] = d;
            mx = fmaxf(mx, d);
        }
    }
    if (tid == 0) {
        float d = 0.0f;
#pragma unroll 8
        for (int i = 0; i < HD; ++i) d = fmaf(qs[i], kns[i], d);
        d *= scale;
        sc[pos] = d;
        mx = fmaxf(mx, d);
    }
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, s));
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int w = 1; w < kAttnThreads / 32; ++w) mx = fmaxf(mx, red[w]);
    __syncthreads();
    float sum = 0.0f;
    for (int t = tid; t <= pos; t += kAttnThreads) {
        const float e = __expf(sc[t] - mx);
        sc[t] = e;
        sum += e;
    }
    sum = block_sum(sum, red);  // ends with a barrier: every sc[] is visible
    // ---- V: thread (slice ks, dims 8 dg .. 8 dg + 7) sums keys ks, ks + KS, ... ----
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0f;
    auto axpy = [&](const uint4& u, float p) {
        const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 f = __bfloat1622float2(e[k]);
            acc[2 * k] = fmaf(p, f.x, acc[2 * k]);
            acc[2 * k + 1] = fmaf(p, f.y, acc[2 * k + 1]);
        }
    };
#pragma unroll
    for (int i = 0; i < VPF; ++i) {
        const int t = ks + i * KS;
        if (t < pos) axpy(vreg[i], sc[t]);
    }
    for (int t = ks + VPF * KS; t < pos; t += 8 * KS) {
        uint4 u[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int tt = t + i * KS;
            u[i] = tt < pos ? __ldg(vp + (long long)tt * DG) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (t + i * KS < pos) axpy(u[i], sc[t + i * KS]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) part[ks][8 * dg + k] = acc[k];
    __syncthreads();
    if (tid < HD) {
        float o = sc[pos] * vns[tid];
#pragma unroll 8
        for (int i = 0; i < KS; ++i) o += part[i][tid];
        att[((long long)b * nh + h) * HD + tid] = __float2bfloat16_rn(o / sum);
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
static cudaError_t launch_pdl_smem(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                   Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
    return launch_pdl_smem(kern, grid, block, 0, s, args...);
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

cudaError_t launch_attn_decode(const void* qkv, const void* cosv, const void* sinv, const float* qn, const float* kn,
                               float eps, void* kc, void* vc, const int* kv_of_q, void* att, int B, int nh, int nkv,
                               int hd, int T, int pos, cudaStream_t s) {
    const size_t smem = sizeof(float) * (pos + 1);
    if (pos < 0 || pos >= T || smem > 200 * 1024) return cudaErrorInvalidValue;
    auto args = [&](auto kern) {
        if (smem > 48 * 1024) {
            const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
        return launch_pdl_smem(kern, dim3(nh, B), dim3(kAttnThreads), smem, s, reinterpret_cast<const __nv_bfloat16*>(qkv),
                          reinterpret_cast<const __nv_bfloat16*>(cosv), reinterpret_cast<const __nv_bfloat16*>(sinv),
                          qn, kn, eps, reinterpret_cast<__nv_bfloat16*>(kc), reinterpret_cast<__nv_bfloat16*>(vc),
                          kv_of_q, reinterpret_cast<__nv_bfloat16*>(att), nh, nkv, T, pos);
    };
    if (hd == 128) return args(k_attn_decode<128>);
    if (hd == 64) return args(k_attn_decode<64>);
    return cudaErrorInvalidValue;
}

cudaError_t launch_silu_mul(const void* gu, void* y, int B, int inter, cudaStream_t s) {
    if (inter % 8) return cudaErrorInvalidValue;
    return launch_pdl(k_silu_mul, dim3(B, (inter / 8 + 255) / 256), dim3(256), s,
                      reinterpret_cast<const __nv_bfloat16*>(gu), reinterpret_cast<__nv_bfloat16*>(y), inter);
}

}  // namespace mq
