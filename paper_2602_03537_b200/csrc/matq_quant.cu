// matq_quant.cu -- the MatGPTQ quantiser's per-weight searches on the GPU
// (SURVEY 8(f) rank 4): every weight scores all 2^c master codes against all
// target bit-widths at once (Alg. 2), the group-scale shrink search, and the
// row-parallel inner column loop of the blocked GPTQ update (Alg. 1).
//
// All arithmetic is float64 with explicit round-to-nearest intrinsics (no FMA
// contraction) in the reference's operation order, so results are bit-identical
// to its numpy code:
//   * select  -- nestquant/gptq.py:104-140 (_select_block / select_codes):
//       err(q) = sum_t lam_t * (w - s * mv_t[q])^2, accumulated over targets in
//       order; argmin with ties to the smallest q;
//   * fit     -- nestquant/grid.py:160-212 (fit_grid): per (row, group) and
//       alpha, q = round_half_away(w / s + z) clipped, obj = sum_t lam_t *
//       pairwise_sum_w (w - s * mv_t[q])^2, where pairwise_sum is numpy's
//       8-accumulator reduction (blocks of <= 128, halves above); first
//       minimum over alpha; scale = max(float32(alpha * base), float32(1e-12));
//   * block   -- nestquant/gptq.py:203-222 (_quantize_columns, within one
//       column block): select on the compensated weight, residual averaged over
//       targets, e = resid / chol[j, j], rank-1 update of the block's later
//       columns.  The update of the columns after the block (Err @ chol) is a
//       plain dgemm left to cuBLAS by the host.
// mv_t[q] = (slice_to_code(q, c, r_t) << (c - r_t)) - 2^(c-1)
// (grid.py:150-157 via slicing.py:31-54), built per CTA in shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "matq_internal.h"

namespace mq {

namespace {

constexpr double kScaleFloor = 1e-12;  // grid.py:20

__device__ __forceinline__ int slice_low(int q, int c, int r) {
    const int k = c - r;
    if (k == 0) return q;
    const int v = (q + (1 << (k - 1))) >> k;
    return v < (1 << r) - 1 ? v : (1 << r) - 1;
}

// shared-memory table mv[t][q] as double, T x 2^c
__device__ __forceinline__ void build_tables(const QuantTargets& tg, double* mv) {
    const int nq = 1 << tg.c, z = 1 << (tg.c - 1);
    for (int i = threadIdx.x; i < tg.T * nq; i += blockDim.x) {
        const int t = i / nq, q = i - t * nq;
        mv[i] = (double)((slice_low(q, tg.c, tg.r[t]) << (tg.c - tg.r[t])) - z);
    }
}

// err(q) for one weight, in the reference's order
__device__ __forceinline__ double cand_err(const QuantTargets& tg, const double* mv, int nq, double w,
                                           double s, int q) {
    double err = 0.0;
    for (int t = 0; t < tg.T; ++t) {
        const double d = __dsub_rn(w, __dmul_rn(s, mv[t * nq + q]));
        err = __dadd_rn(err, __dmul_rn(tg.lam[t], __dmul_rn(d, d)));
    }
    return err;
}

// warp argmin over the 2^c candidates: lanes scan q = lane, lane + 32, ...
// (strict <: first minimum), then (err, q) lexicographic across lanes
__device__ __forceinline__ int warp_select(const QuantTargets& tg, const double* mv, double w, double s) {
    const int nq = 1 << tg.c, lane = threadIdx.x & 31;
    double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    int bq = 0x7fffffff;
    for (int q = lane; q < nq; q += 32) {
        const double e = cand_err(tg, mv, nq, w, s, q);
        if (e < best || bq == 0x7fffffff) {
            best = e;
            bq = q;
        }
    }
#pragma unroll
    for (int sh = 16; sh >= 1; sh >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, sh);
        const int oq = __shfl_xor_sync(0xffffffffu, bq, sh);
        if (oq != 0x7fffffff && (bq == 0x7fffffff || ob < best || (ob == best && oq < bq))) {
            best = ob;
            bq = oq;
        }
    }
    return bq;
}

__global__ void k_select_codes(const double* __restrict__ W, long long ldw, int d_row, int d_col,
                               const float* __restrict__ scales, int ngs, int G, QuantTargets tg,
                               uint8_t* __restrict__ codes, long long ldc) {
    extern __shared__ double mv[];
    build_tables(tg, mv);
    __syncthreads();
    const long long n = (long long)d_row * d_col;
    const long long wpb = blockDim.x >> 5;
    for (long long i = blockIdx.x * wpb + (threadIdx.x >> 5); i < n; i += (long long)gridDim.x * wpb) {
        const int row = (int)(i / d_col), col = (int)(i - (long long)row * d_col);
        const double w = W[row * ldw + col];
        const double s = (double)scales[(long long)row * ngs + col / G];
        const int q = warp_select(tg, mv, w, s);
        if ((threadIdx.x & 31) == 0) codes[row * ldc + col] = (uint8_t)q;
    }
}

// numpy's pairwise sum of a contiguous float64 run (umath loops: blocks of up
// to 128 with 8 accumulators, recursive halving above), single thread
__device__ double pairwise_sum(const double* a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
        return r;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pairwise_sum(a, n2), pairwise_sum(a + n2, n - n2));
}

// the same, a warp at a time for n <= 128: lanes 0..7 own the accumulators
__device__ __forceinline__ double warp_pairwise_sum(const double* a, int n) {
    const int lane = threadIdx.x & 31;
    double res = 0.0;
    if (n > 128 || n < 8) {
        if (lane == 0) res = pairwise_sum(a, n);
    } else {
        const int full = n - (n % 8);
        double r = 0.0;
        if (lane < 8) {
            r = a[lane];
            for (int i = 8 + lane; i < full; i += 8) r = __dadd_rn(r, a[i]);
        }
        const double r1 = __shfl_down_sync(0xffffffffu, r, 1);
        const double p01 = __dadd_rn(r, r1);                        // lanes 0, 2, 4, 6
        const double p23 = __shfl_down_sync(0xffffffffu, p01, 2);
        const double q03 = __dadd_rn(p01, p23);                     // lanes 0, 4
        const double q47 = __shfl_down_sync(0xffffffffu, q03, 4);
        if (lane == 0) {
            res = __dadd_rn(q03, q47);
            for (int i = full; i < n; ++i) res = __dadd_rn(res, a[i]);
        }
    }
    return __shfl_sync(0xffffffffu, res, 0);
}

// one warp per (row, group); smem per warp: G doubles of squared differences + G q's
__global__ void k_fit_grid(const double* __restrict__ W, long long ldw, int d_row, int d_col, int G,
                           QuantTargets tg, const double* __restrict__ alphas, int steps,
                           float* __restrict__ scales, int ngs) {
    extern __shared__ double smem_d[];
    double* mv = smem_d;
    const int nq = 1 << tg.c;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    double* sq = smem_d + tg.T * nq + (size_t)warp * G;
    int* qb = reinterpret_cast<int*>(smem_d + tg.T * nq + (size_t)wpb * G) + (size_t)warp * G;
    build_tables(tg, mv);
    __syncthreads();
    const int z = 1 << (tg.c - 1), qmax = nq - 1;
    const double zmax = (double)((1 << (tg.c - 1)) - 1);
    const long long units = (long long)d_row * ngs;
    for (long long u = (long long)blockIdx.x * wpb + warp; u < units; u += (long long)gridDim.x * wpb) {
        const int row = (int)(u / ngs), g = (int)(u - (long long)row * ngs);
        const int lo = g * G, gw = min(G, d_col - lo);
        const double* wr = W + row * ldw + lo;
        double amax = 0.0;
        for (int k = lane; k < gw; k += 32) amax = fmax(amax, fabs(wr[k]));
#pragma unroll
        for (int sh = 16; sh >= 1; sh >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, sh));
        const double base = fmax(__ddiv_rn(amax, zmax), kScaleFloor);
        double best = 0.0, best_s = 0.0;
        for (int i = 0; i < steps; ++i) {
            const double s = __dmul_rn(alphas[i], base);
            for (int k = lane; k < gw; k += 32) {  // round_half_away(w / s + z), clipped (grid.py:108-111)
                const double x = __dadd_rn(__ddiv_rn(wr[k], s), (double)z);
                const double qr = x >= 0.0 ? floor(__dadd_rn(x, 0.5)) : ceil(__dsub_rn(x, 0.5));
                qb[k] = qr < 0.0 ? 0 : (qr > (double)qmax ? qmax : (int)qr);
            }
            __syncwarp();
            double obj = 0.0;
            for (int t = 0; t < tg.T; ++t) {
                for (int k = lane; k < gw; k += 32) {
                    const double d = __dsub_rn(wr[k], __dmul_rn(s, mv[t * nq + qb[k]]));
                    sq[k] = __dmul_rn(d, d);
                }
                __syncwarp();
                obj = __dadd_rn(obj, __dmul_rn(tg.lam[t], warp_pairwise_sum(sq, gw)));
                __syncwarp();
            }
            if (i == 0 || obj < best) {  // first minimum = the largest alpha
                best = obj;
                best_s = s;
            }
        }
        if (lane == 0) {
            const float f = __double2float_rn(best_s), floor32 = (float)kScaleFloor;
            scales[(long long)row * ngs + g] = f > floor32 ? f : floor32;
        }
    }
}

// Alg. 1 inside one column block [lo, hi): one warp per row (rows are
// independent until the trailing update)
__global__ void k_gptq_block(double* __restrict__ Wc, long long ldw, int d_row, int lo, int hi,
                             const float* __restrict__ scales, int ngs, int G,
                             const double* __restrict__ chol, long long ldch, QuantTargets tg,
                             uint8_t* __restrict__ codes, long long ldc, double* __restrict__ comp,
                             long long ldcomp, double* __restrict__ err, long long lde) {
    extern __shared__ double mv[];
    build_tables(tg, mv);
    __syncthreads();
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const double nt = (double)tg.T;
    const int nq = 1 << tg.c;
    for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < d_row; row += gridDim.x * wpb) {
        double* wrow = Wc + row * ldw;
        for (int j = lo; j < hi; ++j) {
            __syncwarp();
            const double w = wrow[j];
            const double s = (double)scales[(long long)row * ngs + j / G];
            const int q = warp_select(tg, mv, w, s);
            double resid = 0.0;
            for (int t = 0; t < tg.T; ++t) resid = __dadd_rn(resid, __dsub_rn(w, __dmul_rn(s, mv[t * nq + q])));
            resid = __ddiv_rn(resid, nt);
            const double e = __ddiv_rn(resid, chol[(long long)j * ldch + j]);
            if (lane == 0) {
                codes[row * ldc + j] = (uint8_t)q;
                comp[row * ldcomp + j] = w;
                err[row * lde + (j - lo)] = e;
            }
            for (int k = j + 1 + lane; k < hi; k += 32)
                wrow[k] = __dsub_rn(wrow[k], __dmul_rn(e, chol[(long long)j * ldch + k]));
        }
    }
}

int quant_grid(long long units, int wpb) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long want = (units + wpb - 1) / wpb;
    const long long cap = (long long)sms * 8;
    return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

// rtn / round_half_away (grid.py:108-125), elementwise over broadcast operands:
// x = w / s + z (two correctly rounded float64 ops, as numpy), halves away from
// zero, clipped to [0, 2^c - 1] (mode 1) or just rounded (mode 0, round_half_away
// of w itself).  A non-finite w raises flag 1 (rtn's "non-finite weight").
__global__ void k_rtn(const double* __restrict__ w, const double* __restrict__ s, long long n, int c, int mode,
                      double* __restrict__ out_f, long long* __restrict__ out_q, int* __restrict__ err) {
    const double z = (double)(1 << (c - 1)), qmax = (double)((1 << c) - 1);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double wi = w[i];
        if (mode == 0) {
            out_f[i] = wi >= 0.0 ? floor(__dadd_rn(wi, 0.5)) : ceil(__dsub_rn(wi, 0.5));
            continue;
        }
        if (!isfinite(wi)) {
            atomicExch(err, 1);
            out_q[i] = 0;
            continue;
        }
        const double x = __dadd_rn(__ddiv_rn(wi, s[i]), z);
        double q = x >= 0.0 ? floor(__dadd_rn(x, 0.5)) : ceil(__dsub_rn(x, 0.5));
        q = q < 0.0 ? 0.0 : (q > qmax ? qmax : q);  // NaN (0/0 scale) stays NaN -> flag below
        if (q != q) {
            atomicExch(err, 1);
            q = 0.0;
        }
        out_q[i] = (long long)q;
    }
}

}  // namespace

cudaError_t launch_select_codes(const double* W, long long ldw, int d_row, int d_col, const float* scales,
                                int ngs, int G, const QuantTargets& tg, uint8_t* codes, long long ldc,
                                cudaStream_t s) {
    const size_t sm = sizeof(double) * tg.T * ((size_t)1 << tg.c);
    k_select_codes<<<quant_grid((long long)d_row * d_col, 8), 256, sm, s>>>(W, ldw, d_row, d_col, scales, ngs,
                                                                          G, tg, codes, ldc);
    return cudaGetLastError();
}

cudaError_t launch_fit_grid(const double* W, long long ldw, int d_row, int d_col, int G, const QuantTargets& tg,
                            const double* alphas, int steps, float* scales, int ngs, cudaStream_t s) {
    int wpb = 8;
    size_t sm = 0;
    for (;; wpb >>= 1) {
        sm = sizeof(double) * tg.T * ((size_t)1 << tg.c) + (size_t)wpb * G * (sizeof(double) + sizeof(int));
        if (sm <= 200 * 1024 || wpb == 1) break;
    }
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_fit_grid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
    }
    k_fit_grid<<<quant_grid((long long)d_row * ngs, wpb), 32 * wpb, sm, s>>>(W, ldw, d_row, d_col, G, tg, alphas,
                                                                          steps, scales, ngs);
    return cudaGetLastError();
}

cudaError_t launch_gptq_block(double* Wc, long long ldw, int d_row, int lo, int hi, const float* scales, int ngs,
                              int G, const double* chol, long long ldch, const QuantTargets& tg, uint8_t* codes,
                              long long ldc, double* comp, long long ldcomp, double* err, long long lde,
                              cudaStream_t s) {
    const size_t sm = sizeof(double) * tg.T * ((size_t)1 << tg.c);
    k_gptq_block<<<quant_grid(d_row, 4), 128, sm, s>>>(Wc, ldw, d_row, lo, hi, scales, ngs, G, chol, ldch, tg,
                                                     codes, ldc, comp, ldcomp, err, lde);
    return cudaGetLastError();
}

cudaError_t launch_rtn(const double* w, const double* s, long long n, int c, int mode, double* out_f,
                       long long* out_q, int* err, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    k_rtn<<<grid, 256, 0, st>>>(w, s, n, c, mode, out_f, out_q, err);
    return cudaGetLastError();
}

}  // namespace mq
