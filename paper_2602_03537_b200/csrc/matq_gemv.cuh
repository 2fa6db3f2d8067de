// matq_gemv.cuh -- K3: sliced weight-only GEMV / small-batch GEMM, sm_100a.
//
// Y[b, n] = sum_g scale[n, g] * out_scale * sum_{k in g} (s_r(q[n,k]) - 2^(r-1)) * X[b, k]
//
// Replaces the reference's nq_gemv / nq_gemm (packed_kernels.c:84-210, driven
// by kernels/_core.pyx:24-64).  Structure:
//   * Persistent streaming grid: one CTA per SM, sized to use at most half of
//     the SM (registers, shared memory), so that under programmatic dependent
//     launch the NEXT layer's CTAs become resident while this one runs and
//     stream their first weights before waiting on this layer's output.
//   * Work unit = (16-row tile, K chunk of `cs` 256-column steps).  K chunk kc
//     is owned by CTAs with blockIdx % S == kc; each warp walks its units'
//     steps as one flattened sequence, so its TMA ring never drains between
//     row tiles.  Warps are independent: no intra-CTA reduction.
//   * Per step a warp needs one 512-byte slab per plane (the 16 x 256 tile of
//     a plane is contiguous in the P8 layout) plus 128 bytes of group scales;
//     lane 0 keeps `stages` steps in flight with TMA bulk copies
//     (cp.async.bulk + mbarrier complete_tx, L2 evict_first).
//   * Each lane slices its words bitsliced (32 weights per instruction),
//     transposes planes into packed fields, converts them to exact bf16
//     (s - z) already in mma A-fragment order, and feeds mma.m16n8k16 with
//     fp32 accumulation per scale group; activations for the CTA's K chunk
//     are staged once in shared memory and read with ldmatrix.
//   * S == 1: the warp writes Y straight from its accumulators.  S > 1: fp32
//     partials go to a workspace and the last warp to finish a row tile (an
//     atomic ticket per tile) sums them in chunk order -- deterministic, one
//     launch, graph-capturable; tickets return to zero.
#pragma once
#include "matq_common.cuh"

namespace mq {

#ifdef MQ_GEMV_TIMING
// Phase timestamps (globaltimer ns) per (launch slot, CTA, event): profiling builds only.
constexpr int kTsSlots = 64, kTsCtas = 160, kTsEvents = 6;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define MQ_TS(ev) do { if (threadIdx.x == 0 && blockIdx.x < kTsCtas) p.dbg_ts[((size_t)p.dbg_slot * kTsCtas + blockIdx.x) * kTsEvents + (ev)] = gtimer(); } while (0)
#define MQ_TS_MAX(ev) do { if ((threadIdx.x & 31) == 0 && blockIdx.x < kTsCtas) atomicMax(&p.dbg_ts[((size_t)p.dbg_slot * kTsCtas + blockIdx.x) * kTsEvents + (ev)], gtimer()); } while (0)
#else
#define MQ_TS(ev) do { } while (0)
#define MQ_TS_MAX(ev) do { } while (0)
#endif

struct GemvParams {
    const uint32_t* blob;     // step-interleaved blob (parent: 8 planes, child: r planes)
    long long step_words;     // words per (row tile, step) block
    int sb_words;             // scale-block words at the head of each block (16 * spg)
    const float* tscales;     // tiled scales [Np/16][ngp][16] (generic G only)
    const void* X;            // bf16 [B][ldx] or fp32 [B][ldx]
    void* Y;                  // bf16 [B][ldy] or fp32 [B][ldy]
    float* ws;                // fp32 [S][B][Np] when S > 1
    int* tickets;             // [n_rt] zero-initialised, self-resetting
    float out_scale;          // 2^(c - r) for parent slices, 1 for children
    int ldx, ldy;
    int B;                    // logical batch rows
    int Bx;                   // activation rows in the mma N dim (2B when x_f32)
    int N, Np, K, Kp, G, ngp, nsteps, n_rt;
    int S, cs;                // K chunks, steps per chunk
    int ctas_per_chunk;       // gridDim.x / S
    int x_f32;                // X is fp32 (split into hi + lo bf16 rows)
    int y_f32;                // Y is fp32
    int xs_stride;            // smem X row stride (elements)
    int xcopy_stride;         // elements between activation copies (zero-point folding)
    int cs_off;               // smem byte offset of the per-group zero-point constants
    int xs_bytes;             // smem bytes of the X staging area (16-aligned)
    int stages;               // per-warp TMA ring depth (<= 8)
    int pair;                 // S == 2 on CTA pairs (clusters of 2): chunk 1 ships partials by st.async
    int pair_off;             // smem byte offset of [warps x pair_units mbarriers][slots]
    int pair_units;           // most row tiles a warp holds
    int dbg_slot;             // MQ_GEMV_TIMING builds: timestamp slot of this launch
    unsigned long long* dbg_ts;
};

#ifndef MQ_GEMV_DEBUG
#define MQ_GEMV_DEBUG 0  // profiling builds: 1 = skip decode, 2 = skip weight loads
#endif

#ifndef MQ_GEMV_MAX_WARPS
#define MQ_GEMV_MAX_WARPS 16
#endif
constexpr int kMaxWarps = MQ_GEMV_MAX_WARPS;

template <int R, int NT, bool CHILD, int GS>
__global__ void __launch_bounds__(NT >= 4 ? 256 : kMaxWarps * 32, 1) k_gemv(const GemvParams p) {
    constexpr int NPL = PlaneCount<R, CHILD>::value;
    constexpr uint32_t kSlab = 512;
    constexpr uint32_t kScaleBytes = GS == 128 ? 128 : 0;   // 2 groups x 16 rows, head of block
    constexpr uint32_t kStageBytes = kScaleBytes + NPL * kSlab;
    // zero-point folding (zp_off<R>, matq_common.cuh): raw magic-encoded A + scaled activation copies
    // zero-point folding only for NT == 1 (B <= 8): its scaled activation copies
    // multiply the staging by 2-3x, which at larger B forces tiny K chunks and
    // heavy split-K; there the exact HFMA2 decode (idle FMA pipe) is cheaper
    constexpr bool ZP = (GS == 128) && (R != 8) && (NT == 1) && !(MQ_GEMV_DEBUG & 1);
    constexpr int NCOPY = ZP ? zp_ncopies(R) : 1;
    extern __shared__ __align__(16) uint8_t smem[];
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem);

    const int nwarps = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int kc = blockIdx.x % p.S, j = blockIdx.x / p.S;
    const int chunk0 = kc * p.cs;
    const int ns = max(0, min(chunk0 + p.cs, p.nsteps) - chunk0);
    // row tiles dealt warp-major across the chunk's CTAs, so every SM gets work
    const int rt_first = warp * p.ctas_per_chunk + j;
    const int rt_stride = p.ctas_per_chunk * nwarps;
    const int n_units = (rt_first < p.n_rt && ns > 0) ? (p.n_rt - 1 - rt_first) / rt_stride + 1 : 0;
    const int total = n_units * ns;  // flattened (unit, step) sequence of this warp

    // ---- per-warp TMA ring --------------------------------------------------
    const int D = p.stages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.xs_bytes);
    uint8_t* ring = smem + p.xs_bytes + kMaxWarps * 8 * 8;
    const uint32_t my_bar0 = smem_addr(bars + warp * 8);
    const uint32_t my_ring0 = smem_addr(ring + (size_t)warp * D * kStageBytes);
    uint64_t policy = 0;
    if (lane == 0) {
        policy = policy_evict_first();
        for (int i = 0; i < D; ++i) mbar_init(my_bar0 + 8 * i, 1);
        fence_mbar_init();
    }
    __syncwarp();
    // One bulk copy per step: [scales][planes 0..NPL-1] are contiguous at the
    // head of the (rt, st) block.  The issue cursor advances incrementally.
    const uint32_t skip_words = (uint32_t)(p.sb_words - kScaleBytes / 4);  // scale words not needed
    const uint32_t* issue_ptr = p.blob + ((long long)rt_first * p.nsteps + chunk0) * p.step_words + skip_words;
    int issue_li = 0, issue_stage = 0;
    const long long unit_jump = ((long long)rt_stride * p.nsteps - ns) * p.step_words;
    auto issue_next = [&]() {  // lane 0 only
        const uint32_t bar = my_bar0 + 8 * issue_stage;
        mbar_expect_tx(bar, kStageBytes);
        bulk_g2s(my_ring0 + issue_stage * kStageBytes, issue_ptr, kStageBytes, bar, policy);
        issue_ptr += p.step_words;
        if (++issue_li == ns) {
            issue_li = 0;
            issue_ptr += unit_jump;
        }
        if (++issue_stage == D) issue_stage = 0;
    };
    // Weights do not depend on the previous kernel: fill the ring before
    // waiting on the programmatic dependency (X, workspace, Y).
    if (lane == 0 && !(MQ_GEMV_DEBUG & 2))
        for (int i = 0; i < D && i < total; ++i) issue_next();
    MQ_TS(0);
    pdl_launch_dependents();
    pdl_wait();
    MQ_TS(1);

    // ---- stage X[:, chunk columns] into shared memory as bf16 rows ----------
    // copy c (ZP only) holds x * 2^-zp_copy_off(R, c): exact power-of-two scaling.
    const int Kc = p.cs * kStepCols;
    const int col_base = chunk0 * kStepCols;
    auto put = [&](int row, int c, uint16_t v) {
        xs[row * p.xs_stride + c] = v;
        if constexpr (NCOPY > 1) {
#pragma unroll
            for (int cp = 1; cp < NCOPY; ++cp) {
                const float f = bf16_to_f32(v) * (1.0f / (float)(1 << zp_copy_off(R, cp)));
                xs[cp * p.xcopy_stride + row * p.xs_stride + c] = f32_to_bf16_rn(f);
            }
        }
    };
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
                if constexpr (NCOPY > 1) {
                    const uint16_t* hv = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
                    for (int cp = 1; cp < NCOPY; ++cp) {
                        uint4 o;
                        uint16_t* ho = reinterpret_cast<uint16_t*>(&o);
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            ho[e] = f32_to_bf16_rn(bf16_to_f32(hv[e]) * (1.0f / (float)(1 << zp_copy_off(R, cp))));
                        *reinterpret_cast<uint4*>(xs + cp * p.xcopy_stride + b * p.xs_stride + c) = o;
                    }
                }
            }
        } else {
            for (int idx = threadIdx.x; idx < p.B * Kc; idx += blockDim.x) {
                const int b = idx / Kc, c = idx - b * Kc;
                const int col = col_base + c;
                put(b, c, col < p.K ? X[(long long)b * p.ldx + col] : (uint16_t)0);
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
            put(2 * b, c, hi);
            put(2 * b + 1, c, lo);
        }
    }
    if (p.pair && lane == 0) {  // chunk 0's per-(warp, unit) barriers (used once per launch)
        const uint32_t pb = smem_addr(smem + p.pair_off);
        for (int u = 0; u < p.pair_units; ++u) mbar_init(pb + 8 * (warp * p.pair_units + u), 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (p.pair) cluster_sync_all();  // the peer's st.async lands on initialised barriers
    MQ_TS(2);

    // ldmatrix row addresses: matrix mi = lane >> 3 covers k offset 8*mi of a
    // 32-column pair of k16 steps; row n = nt*8 + (lane & 7) (rows >= Bx read
    // row 0: their outputs are discarded).
    // With ZP, matrix mi = (k16 step s = 2*s2 + (mi >> 1), half mi & 1) reads the
    // activation copy matching that half's field offset.
    const uint32_t xs_saddr = smem_addr(xs);
    uint32_t xrow_addr[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        int n = nt * 8 + (lane & 7);
        if (n >= p.Bx) n = 0;
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int mi = lane >> 3;
            int cp = 0;
            if constexpr (ZP) {
                const int sx = 2 * s2 + (mi >> 1), hx = mi & 1;
                cp = zp_copy_of(R, zp_off<R>(sx, hx));
            }
            xrow_addr[nt][s2] =
                xs_saddr + (uint32_t)(cp * p.xcopy_stride + n * p.xs_stride + 8 * mi) * 2u;
        }
    }
    // Per-group zero-point constants: the same MMA chain as a group of the
    // main loop, on the all-zero-code fragment, once per CTA.
    float* zc = reinterpret_cast<float*>(smem + p.cs_off);
    if constexpr (ZP) {
        const int ngc = 2 * p.cs;
        for (int gi = warp; gi < ngc; gi += nwarps) {
            float cacc[NT][4];
#pragma unroll
            for (int w2 = 0; w2 < 2; ++w2)
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    uint32_t bf[NT][4];
                    const uint32_t xcol = (uint32_t)(gi * 128 + 64 * w2 + 32 * s2);
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) ldmatrix_x4(bf[nt], xrow_addr[nt][s2] + xcol * 2u);
#pragma unroll
                    for (int sh = 0; sh < 2; ++sh) {
                        const int s = 2 * s2 + sh;
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) {
                            if (w2 == 0 && s == 0)
                                mma_zero(cacc[nt], zp_zero_a<R>(s, 0), zp_zero_a<R>(s, 1), zp_zero_a<R>(s, 2),
                                         zp_zero_a<R>(s, 3), bf[nt][2 * sh], bf[nt][2 * sh + 1]);
                            else
                                mma_acc(cacc[nt], zp_zero_a<R>(s, 0), zp_zero_a<R>(s, 1), zp_zero_a<R>(s, 2),
                                        zp_zero_a<R>(s, 3), bf[nt][2 * sh], bf[nt][2 * sh + 1]);
                        }
                    }
                }
            if (g == 0) {
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    zc[gi * (NT * 8) + nt * 8 + 2 * t] = cacc[nt][0];
                    zc[gi * (NT * 8) + nt * 8 + 2 * t + 1] = cacc[nt][1];
                }
            }
        }
        __syncthreads();
    }
    MQ_TS(3);

    float tot[NT][4];
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) tot[nt][i] = 0.0f, acc[nt][i] = 0.0f;

    // generic group size bookkeeping (GS == 0): groups may straddle steps
    int next_bound = 0, cur_grp = 0, cur_rt = 0;
    auto flush_generic = [&]() {
        const float* sp = p.tscales + ((long long)cur_rt * p.ngp + cur_grp) * 16 + g;
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
            for (int jj = 0; jj < NPL; ++jj) T[jj] = word_of(buf[jj], w);
            uint32_t A[16];
            if (MQ_GEMV_DEBUG & 1) {
#pragma unroll
                for (int q = 0; q < 16; ++q) A[q] = T[q % NPL] & 0x3F3F3F3Fu;
            } else {
                uint32_t S[R];
                slice_loaded<R, CHILD>(T, S);
                decode_word<R, ZP>(S, A);
            }
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                uint32_t bf[NT][4];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    ldmatrix_x4(bf[nt], xrow_addr[nt][s2] + (xcol + 64 * w + 32 * s2) * 2u);
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
                        if constexpr (ZP) {
                            const float* zp = zc + ((int)(xcol >> 7) + (w >> 1)) * (NT * 8) + nt * 8 + 2 * t;
                            const float c0 = zp[0], c1 = zp[1];
                            tot[nt][0] = fmaf(s_lo, acc[nt][0] - c0, tot[nt][0]);
                            tot[nt][1] = fmaf(s_lo, acc[nt][1] - c1, tot[nt][1]);
                            tot[nt][2] = fmaf(s_hi, acc[nt][2] - c0, tot[nt][2]);
                            tot[nt][3] = fmaf(s_hi, acc[nt][3] - c1, tot[nt][3]);
                        } else {
                            tot[nt][0] = fmaf(s_lo, acc[nt][0], tot[nt][0]);
                            tot[nt][1] = fmaf(s_lo, acc[nt][1], tot[nt][1]);
                            tot[nt][2] = fmaf(s_hi, acc[nt][2], tot[nt][2]);
                            tot[nt][3] = fmaf(s_hi, acc[nt][3], tot[nt][3]);
                        }
                    }
                }
            }
        }
    };

    // Output element (b, row) held by this thread for accumulator (nt, i):
    // row = 16 rt + g + 8 (i >> 1), mma column n = 8 nt + 2 t + (i & 1);
    // plain X: b = n; split X: columns (2b, 2b+1) = (hi, lo) of b = 4 nt + t.
    auto store_y = [&](int b, int row, float v) {
        if (p.y_f32)
            reinterpret_cast<float*>(p.Y)[(long long)b * p.ldy + row] = v;
        else
            reinterpret_cast<uint16_t*>(p.Y)[(long long)b * p.ldy + row] = f32_to_bf16_rn(v);
    };
    int unit_idx = 0;  // this warp's finished tiles (pair slot index)
    auto finalize = [&](int rt) {
        MQ_TS_MAX(5);
        if constexpr (GS == 0) flush_generic();
        const int r0 = rt * kTileRows + g;
        float v[NT][2][2];  // [nt][row half][column parity | hi+lo combined]
        int bcol[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            if (!p.x_f32) {
                v[nt][0][0] = tot[nt][0] * p.out_scale;
                v[nt][0][1] = tot[nt][1] * p.out_scale;
                v[nt][1][0] = tot[nt][2] * p.out_scale;
                v[nt][1][1] = tot[nt][3] * p.out_scale;
                bcol[nt][0] = nt * 8 + 2 * t;
                bcol[nt][1] = nt * 8 + 2 * t + 1;
            } else {
                v[nt][0][0] = (tot[nt][0] + tot[nt][1]) * p.out_scale;
                v[nt][1][0] = (tot[nt][2] + tot[nt][3]) * p.out_scale;
                v[nt][0][1] = v[nt][1][1] = 0.0f;
                bcol[nt][0] = nt * 4 + t;
                bcol[nt][1] = 1 << 30;  // no second column
            }
        }
        if (p.S == 1) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int row = r0 + 8 * h, b = bcol[nt][c];
                        if (b < p.B && row < p.N) store_y(b, row, v[nt][h][c]);
                    }
            return;
        }
        if (p.pair) {
            // chunk 1 ships its partial into chunk 0's slot; chunk 0 adds it (chunk order)
            const int ui = unit_idx++;
            const uint32_t pb = smem_addr(smem + p.pair_off);
            const uint32_t bar = pb + 8 * (warp * p.pair_units + ui);
            const uint32_t slot = pb + ((8u * (uint32_t)(kMaxWarps * p.pair_units) + 15u) & ~15u) +
                                  (uint32_t)(((warp * p.pair_units + ui) * 32 + lane) * NT * 16);
            if (kc == 1) {
                const uint32_t rbar = mapa_rank(bar, 0), rslot = mapa_rank(slot, 0);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    st_async_v4(rslot + 16 * nt, v[nt][0][0], v[nt][0][1], v[nt][1][0], v[nt][1][1], rbar);
                return;
            }
            if (lane == 0) mbar_expect_tx(bar, 32u * NT * 16u);
            __syncwarp();
            mbar_wait(bar, 0);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const uint4 q = lds128(slot + 16 * nt);
                const float pv[2][2] = {{__uint_as_float(q.x), __uint_as_float(q.y)},
                                        {__uint_as_float(q.z), __uint_as_float(q.w)}};
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int row = r0 + 8 * h, b = bcol[nt][c];
                        if (b < p.B && row < p.N) store_y(b, row, v[nt][h][c] + pv[h][c]);
                    }
            }
            return;
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int row = r0 + 8 * h, b = bcol[nt][c];
                    if (b < p.B && row < p.N)
                        p.ws[((long long)kc * p.B + b) * p.Np + row] = v[nt][h][c];
                }
        // publish: warp barrier orders all lanes' partials before lane 0's
        // release-RMW on the tile ticket; the last arriver acquires.
        __syncwarp();
        int last = 0;
        // lane 1, not lane 0: lane 0 issues the ring's bulk copies, and an acq_rel
        // RMW would wait for those in-flight loads to land
        if (lane == 1) last = (atom_add_acq_rel(p.tickets + rt, 1) == p.S - 1);
        last = __shfl_sync(0xffffffffu, last, 1);
        if (!last) return;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int row = r0 + 8 * h, b = bcol[nt][c];
                    if (b < p.B && row < p.N) {
                        const float* wp = p.ws + (long long)b * p.Np + row;
                        const long long cstride = (long long)p.B * p.Np;
                        float s = 0.0f;
                        int q = 0;
                        for (; q + 4 <= p.S; q += 4) {  // independent loads, ordered sum
                            const float a0 = __ldcg(wp + q * cstride), a1 = __ldcg(wp + (q + 1) * cstride);
                            const float a2 = __ldcg(wp + (q + 2) * cstride), a3 = __ldcg(wp + (q + 3) * cstride);
                            s += a0; s += a1; s += a2; s += a3;
                        }
                        for (; q < p.S; ++q) s += __ldcg(wp + q * cstride);
                        store_y(b, row, s);
                    }
                }
        __syncwarp();
        if (lane == 0) p.tickets[rt] = 0;
    };

    int li = 0, stage = 0, rt = rt_first;
    uint32_t parity = 0;
#pragma unroll 1
    for (int f = 0; f < total; ++f) {
        const int st = chunk0 + li;
        if (li == 0) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < 4; ++i) tot[nt][i] = 0.0f;
            if constexpr (GS == 0) {
                cur_rt = rt;
                cur_grp = (st * kStepCols) / p.G;
                next_bound = (cur_grp + 1) * p.G;
            }
        }
        if (!(MQ_GEMV_DEBUG & 2)) mbar_wait(my_bar0 + 8 * stage, parity);
        const uint32_t src = my_ring0 + stage * kStageBytes;
        float sc[4];
        if constexpr (GS == 128) {
            sc[0] = lds32f(src + g * 4);
            sc[1] = lds32f(src + (g + 8) * 4);
            sc[2] = lds32f(src + (16 + g) * 4);
            sc[3] = lds32f(src + (24 + g) * 4);
        }
        uint4 buf[NPL];
#pragma unroll
        for (int jj = 0; jj < NPL; ++jj) buf[jj] = lds128(src + kScaleBytes + jj * kSlab + lane * 16);
        __syncwarp();
        if (lane == 0 && f + D < total && !(MQ_GEMV_DEBUG & 2)) {
            fence_proxy_async_smem();
            issue_next();
        }
        process(buf, sc, st);
        if (++li == ns) {
            finalize(rt);
            li = 0;
            rt += rt_stride;
        }
        if (++stage == D) {
            stage = 0;
            parity ^= 1u;
        }
    }
    MQ_TS_MAX(4);
}

// Host-side launcher table entry, implemented per R in matq_gemv_r*.cu.
using GemvLaunchFn = cudaError_t (*)(const GemvParams&, int nt, bool child, int gs, dim3 grid,
                                     dim3 block, size_t smem, cudaStream_t stream, bool pdl);

template <int R>
cudaError_t launch_gemv_r(const GemvParams& p, int nt, bool child, int gs, dim3 grid, dim3 block,
                          size_t smem, cudaStream_t stream, bool pdl);

}  // namespace mq
