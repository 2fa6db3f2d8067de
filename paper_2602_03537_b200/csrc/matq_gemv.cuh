// matq_gemv.cuh -- K3: sliced weight-only GEMV / small-batch GEMM, sm_100a.
//
// Y[b, n] = sum_g scale[n, g] * out_scale * sum_{k in g} (s_r(q[n,k]) - 2^(r-1)) * X[b, k]
//
// This replaces the reference's nq_gemv / nq_gemm (packed_kernels.c:84-210,
// driven by kernels/_core.pyx:24-64).  Work decomposition:
//   * a warp owns one 16-row tile and a contiguous run of 256-column steps;
//   * per step it needs one 512-byte slab per plane (the 16 x 256 tile of
//     that plane is contiguous) plus 128 bytes of group scales; lane 0 of
//     each warp keeps a ring of `stages` such steps in flight with TMA bulk
//     copies (cp.async.bulk + mbarrier complete_tx, L2 evict_first), so the
//     memory pipeline costs no registers and one instruction per slab;
//   * each lane slices its words bitsliced (32 weights / op), transposes the
//     planes into packed fields and converts them to exact bf16 (s - z) in
//     registers, already in mma A-fragment order (the P8 layout guarantees
//     it), and feeds mma.m16n8k16 with fp32 accumulation per scale group;
//   * X for the CTA's column range is staged once in shared memory and read
//     as B fragments with ldmatrix;
//   * warps of a CTA split K and reduce through shared memory in fixed
//     order; CTAs that split K further write fp32 partials to a workspace
//     and the last CTA to arrive (atomic ticket) reduces them in split order
//     -- deterministic, one launch, graph-capturable.
#pragma once
#include "matq_common.cuh"

namespace mq {

struct GemvParams {
    const uint32_t* planes;   // P8 planes (parent) or child planes
    long long plane_stride;   // uint32 words between consecutive planes
    const float* tscales;     // tiled scales [Np/16][ngp][16]
    const void* X;            // bf16 [B][ldx] or fp32 [B][ldx]
    void* Y;                  // bf16 [B][ldy] or fp32 [B][ldy]
    float* ws;                // fp32 [S][B][Np] when S > 1
    int* tickets;             // [gridDim.x] zero-initialised, self-resetting
    float out_scale;          // 2^(c - r) for parent slices, 1 for children
    int ldx, ldy;
    int B;                    // logical batch rows
    int Bx;                   // activation rows in the mma N dim (2B when x_split)
    int N, Np, K, Kp, G, ngp, nsteps;
    int RT, KW, ITERS, S;     // decomposition (see choose_gemv_config)
    int x_f32;                // X is fp32 (split into hi + lo bf16 rows)
    int y_f32;                // Y is fp32
    int xs_stride;            // smem X row stride (elements)
    int stages;               // per-warp TMA ring depth
    int xs_bytes;             // smem bytes reserved for X staging / reduction (16-aligned)
};

template <int R, int NT, bool CHILD, int GS>
__global__ void __launch_bounds__(256, NT >= 4 ? 1 : 2) k_gemv(const GemvParams p) {
    constexpr int NPL = PlaneCount<R, CHILD>::value;
    extern __shared__ __align__(16) uint8_t smem[];
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2;
    const int rt_l = warp % p.RT, ks = warp / p.RT;
    const int n_rt = p.Np / kTileRows;
    const int rt = blockIdx.x * p.RT + rt_l;
    const int split = blockIdx.y;
    const int cta_step0 = split * p.KW * p.ITERS;
    const int st0 = cta_step0 + ks * p.ITERS;
    const int st1 = min(st0 + p.ITERS, p.nsteps);
    const bool has_work = rt < n_rt && st0 < st1;

    const float* sbase = p.tscales + (long long)(has_work ? rt : 0) * p.ngp * 16;

    // ---- per-warp TMA bulk ring: stage = NPL plane slabs (512 B) + scales --
    constexpr uint32_t kSlab = 512;
    constexpr uint32_t kScaleBytes = GS == 128 ? 128 : 0;
    constexpr uint32_t kStageBytes = NPL * kSlab + kScaleBytes;
    const int D = p.stages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.xs_bytes);
    uint8_t* ring = smem + p.xs_bytes + 8 * 8 * 8;  // 8 warps x up to 8 stages x 8 B
    const uint32_t my_bar0 = smem_addr(bars + warp * 8);
    const uint32_t my_ring0 = smem_addr(ring + (size_t)warp * D * kStageBytes);
    const uint32_t* gplanes = p.planes + ((long long)(has_work ? rt : 0) * p.nsteps) * 128;
    const float* gscales = sbase;
    uint64_t policy = 0;
    if (lane == 0) {
        policy = policy_evict_first();
        for (int i = 0; i < D; ++i) mbar_init(my_bar0 + 8 * i, 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int st, int stage) {  // lane 0 only
        const uint32_t bar = my_bar0 + 8 * stage;
        const uint32_t dst = my_ring0 + stage * kStageBytes;
        mbar_expect_tx(bar, kStageBytes);
#pragma unroll
        for (int j = 0; j < NPL; ++j)
            bulk_g2s(dst + j * kSlab, gplanes + j * p.plane_stride + (long long)st * 128, kSlab, bar,
                     policy);
        if constexpr (GS == 128) bulk_g2s(dst + NPL * kSlab, gscales + (2 * st) * 16, kScaleBytes, bar, policy);
    };
    // Weights do not depend on the previous kernel: fill the ring before
    // waiting on the programmatic dependency (X / workspace).
    if (has_work && lane == 0)
        for (int i = 0; i < D && st0 + i < st1; ++i) issue(st0 + i, i);
    pdl_launch_dependents();
    pdl_wait();

    // ---- stage X[:, cta columns] into shared memory as bf16 rows ----------
    const int Kc = p.KW * p.ITERS * kStepCols;
    const int col_base = cta_step0 * kStepCols;
    if (!p.x_f32) {
        const uint16_t* X = reinterpret_cast<const uint16_t*>(p.X);
        const bool vec = ((p.ldx & 7) == 0) && ((p.K & 7) == 0) &&
                         ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
        if (vec) {
            const int c8 = Kc >> 3;
            for (int idx = threadIdx.x; idx < p.B * c8; idx += blockDim.x) {
                const int b = idx / c8, c = (idx - b * c8) * 8;
                const int col = col_base + c;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (col < p.K) v = __ldg(reinterpret_cast<const uint4*>(X + (long long)b * p.ldx + col));
                *reinterpret_cast<uint4*>(xs + b * p.xs_stride + c) = v;
            }
        } else {
            for (int idx = threadIdx.x; idx < p.B * Kc; idx += blockDim.x) {
                const int b = idx / Kc, c = idx - b * Kc;
                const int col = col_base + c;
                xs[b * p.xs_stride + c] = col < p.K ? X[(long long)b * p.ldx + col] : (uint16_t)0;
            }
        }
    } else {
        // fp32 activations: x = hi + lo with hi = bf16(x), lo = bf16(x - hi);
        // rows 2b / 2b+1 so one thread's accumulator pair holds both halves.
        const float* X = reinterpret_cast<const float*>(p.X);
        for (int idx = threadIdx.x; idx < p.B * Kc; idx += blockDim.x) {
            const int b = idx / Kc, c = idx - b * Kc;
            const int col = col_base + c;
            const float x = col < p.K ? X[(long long)b * p.ldx + col] : 0.0f;
            const uint16_t hi = f32_to_bf16_rn(x);
            const uint16_t lo = f32_to_bf16_rn(x - bf16_to_f32(hi));
            xs[(2 * b) * p.xs_stride + c] = hi;
            xs[(2 * b + 1) * p.xs_stride + c] = lo;
        }
    }
    __syncthreads();

    // ldmatrix row addresses: matrix mi = lane >> 3 covers k offset 8*mi of a
    // 32-column pair of k16 steps; row n = nt*8 + (lane & 7) (rows >= Bx read
    // row 0: their outputs are discarded).
    const uint32_t xs_saddr = static_cast<uint32_t>(__cvta_generic_to_shared(xs));
    uint32_t xrow_addr[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        int n = nt * 8 + (lane & 7);
        if (n >= p.Bx) n = 0;
        xrow_addr[nt] = xs_saddr + (uint32_t)(n * p.xs_stride + 8 * (lane >> 3)) * 2u;
    }

    float tot[NT][4];
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) tot[nt][i] = 0.0f, acc[nt][i] = 0.0f;

    // generic group size bookkeeping (GS == 0)
    int next_bound = 0, cur_grp = 0;
    if constexpr (GS == 0) {
        const int c0 = st0 * kStepCols;
        cur_grp = c0 / p.G;
        next_bound = (cur_grp + 1) * p.G;
    }

    auto flush_generic = [&]() {
        const float* sp = sbase + cur_grp * 16 + g;
        const float s_lo = __ldg(sp), s_hi = __ldg(sp + 8);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            tot[nt][0] = fmaf(s_lo, acc[nt][0], tot[nt][0]);
            tot[nt][1] = fmaf(s_lo, acc[nt][1], tot[nt][1]);
            tot[nt][2] = fmaf(s_hi, acc[nt][2], tot[nt][2]);
            tot[nt][3] = fmaf(s_hi, acc[nt][3], tot[nt][3]);
            acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.0f;
        }
    };

    auto process = [&](const uint4 (&buf)[NPL], const float (&sc)[4], int st) {
        const uint32_t xcol = (uint32_t)(st * kStepCols - col_base);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            uint32_t T[NPL];
#pragma unroll
            for (int j = 0; j < NPL; ++j) T[j] = word_of(buf[j], w);
            uint32_t S[R];
            slice_loaded<R, CHILD>(T, S);
            uint32_t A[16];
            decode_word<R>(S, A);
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                uint32_t bf[NT][4];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    ldmatrix_x4(bf[nt], xrow_addr[nt] + (xcol + 64 * w + 32 * s2) * 2u);
#pragma unroll
                for (int sh = 0; sh < 2; ++sh) {
                    const int s = 2 * s2 + sh;
                    if constexpr (GS == 0) {
                        const int gc = st * kStepCols + 64 * w + 16 * s;
                        if (gc == next_bound) {
                            flush_generic();
                            cur_grp = gc / p.G;
                            next_bound = (cur_grp + 1) * p.G;
                        }
                    }
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        if constexpr (GS == 128) {
                            if ((w & 1) == 0 && s == 0)
                                mma_zero(acc[nt], A[4 * s], A[4 * s + 1], A[4 * s + 2], A[4 * s + 3],
                                         bf[nt][2 * sh], bf[nt][2 * sh + 1]);
                            else
                                mma_acc(acc[nt], A[4 * s], A[4 * s + 1], A[4 * s + 2], A[4 * s + 3],
                                        bf[nt][2 * sh], bf[nt][2 * sh + 1]);
                        } else {
                            mma_acc(acc[nt], A[4 * s], A[4 * s + 1], A[4 * s + 2], A[4 * s + 3],
                                    bf[nt][2 * sh], bf[nt][2 * sh + 1]);
                        }
                    }
                }
            }
            if constexpr (GS == 128) {
                if (w & 1) {
                    const float s_lo = sc[(w >> 1) * 2], s_hi = sc[(w >> 1) * 2 + 1];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        tot[nt][0] = fmaf(s_lo, acc[nt][0], tot[nt][0]);
                        tot[nt][1] = fmaf(s_lo, acc[nt][1], tot[nt][1]);
                        tot[nt][2] = fmaf(s_hi, acc[nt][2], tot[nt][2]);
                        tot[nt][3] = fmaf(s_hi, acc[nt][3], tot[nt][3]);
                    }
                }
            }
        }
    };

    if (has_work) {
#pragma unroll 1
        for (int i = 0, st = st0; st < st1; ++i, ++st) {
            const int stage = i % D;
            mbar_wait(my_bar0 + 8 * stage, (uint32_t)((i / D) & 1));
            const uint32_t src = my_ring0 + stage * kStageBytes;
            uint4 buf[NPL];
#pragma unroll
            for (int j = 0; j < NPL; ++j) buf[j] = lds128(src + j * kSlab + lane * 16);
            float sc[4];
            if constexpr (GS == 128) {
                sc[0] = lds32f(src + NPL * kSlab + g * 4);
                sc[1] = lds32f(src + NPL * kSlab + (g + 8) * 4);
                sc[2] = lds32f(src + NPL * kSlab + (16 + g) * 4);
                sc[3] = lds32f(src + NPL * kSlab + (24 + g) * 4);
            }
            __syncwarp();
            if (lane == 0 && st + D < st1) {
                fence_proxy_async_smem();
                issue(st + D, stage);
            }
            process(buf, sc, st);
        }
        if constexpr (GS == 0) flush_generic();
    }

    // ---- epilogue: fixed-order reduction over the CTA's K warps ------------
    __syncthreads();  // X staging area is reused as the reduction buffer
    float* red = reinterpret_cast<float*>(smem);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) red[((warp * NT + nt) * 4 + i) * 32 + lane] = tot[nt][i];
    __syncthreads();

    const int rows_cta = p.RT * kTileRows;
    const int row0 = blockIdx.x * rows_cta;
    const bool multi = p.S > 1;
    for (int idx = threadIdx.x; idx < p.B * rows_cta; idx += blockDim.x) {
        const int b = idx / rows_cta, rl = idx - b * rows_cta;
        const int rtl = rl >> 4, r16 = rl & 15;
        const int gg = r16 & 7, hi = r16 >> 3;
        float v = 0.0f;
        if (!p.x_f32) {
            const int nt = b >> 3, cc = b & 7;
            const int ln = gg * 4 + (cc >> 1), i = hi * 2 + (cc & 1);
            for (int k2 = 0; k2 < p.KW; ++k2) v += red[(((k2 * p.RT + rtl) * NT + nt) * 4 + i) * 32 + ln];
        } else {
            const int c = 2 * b, nt = c >> 3, cc = c & 7;
            const int ln = gg * 4 + (cc >> 1), i = hi * 2;
            float vh = 0.0f, vl = 0.0f;
            for (int k2 = 0; k2 < p.KW; ++k2) {
                const float* rp = red + (((k2 * p.RT + rtl) * NT + nt) * 4 + i) * 32 + ln;
                vh += rp[0];
                vl += rp[32];
            }
            v = vh + vl;
        }
        v *= p.out_scale;
        const int row = row0 + rl;
        if (multi) {
            p.ws[((long long)split * p.B + b) * p.Np + row] = v;
        } else if (row < p.N) {
            if (p.y_f32)
                reinterpret_cast<float*>(p.Y)[(long long)b * p.ldy + row] = v;
            else
                reinterpret_cast<uint16_t*>(p.Y)[(long long)b * p.ldy + row] = f32_to_bf16_rn(v);
        }
    }
    if (!multi) return;

    // ---- cross-CTA split-K: last CTA to arrive reduces in split order -------
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(p.tickets + blockIdx.x, 1);
        s_last = (prev == p.S - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int idx = threadIdx.x; idx < p.B * rows_cta; idx += blockDim.x) {
        const int b = idx / rows_cta, rl = idx - b * rows_cta;
        const int row = row0 + rl;
        if (row >= p.N) continue;
        float v = 0.0f;
        for (int s = 0; s < p.S; ++s) v += __ldcg(p.ws + ((long long)s * p.B + b) * p.Np + row);
        if (p.y_f32)
            reinterpret_cast<float*>(p.Y)[(long long)b * p.ldy + row] = v;
        else
            reinterpret_cast<uint16_t*>(p.Y)[(long long)b * p.ldy + row] = f32_to_bf16_rn(v);
    }
    if (threadIdx.x == 0) p.tickets[blockIdx.x] = 0;
}

// Host-side launcher table entry, implemented per R in matq_gemv_r*.cu.
using GemvLaunchFn = cudaError_t (*)(const GemvParams&, int nt, bool child, int gs, dim3 grid,
                                     size_t smem, cudaStream_t stream, bool pdl);

template <int R>
cudaError_t launch_gemv_r(const GemvParams& p, int nt, bool child, int gs, dim3 grid, size_t smem,
                          cudaStream_t stream, bool pdl);

}  // namespace mq
