// matq_gemm.cuh -- K4: prefill dequant-GEMM on the 5th-generation tensor cores.
//
// Y[b, n] = sum_k X[b, k] * scale[n, k / 128] * out_scale * (s_r(q[n, k]) - 2^(r-1))
// for token counts past the GEMV range (B > 32; BASELINE config C4).  The
// reference has no batched GPU path; its CPU analogue is nq_gemm
// (packed_kernels.c:177-210, driven in chunks of 16 rows by
// kernels/_core.pyx:53-63).
//
// Persistent CTAs (one per SM, 23 warps).  Work unit = (output tile of 128
// weight rows x BN tokens, K split).  Pipelines:
//   raw ring    warp 2 (one lane) bulk-copies, per 256-column step, the eight
//               16-row P8 blocks of the tile ([group scales][r+1 plane slabs],
//               each contiguous) into shared memory (TMA, mbarrier complete_tx);
//               it does not wait on the previous kernel (weights are static)
//   operand     per 64-column stage: A = 128 x 64 bf16 weights, B = BN x 64
//   stages      bf16 activations, both K-major SWIZZLE_128B; warp 0 (one lane)
//               TMA-loads B from a tensor map (zero fill past B and K) after the
//               programmatic-dependency wait; warps 7-22 decode (one 16-row
//               block x one word pair each): slice + decode bitsliced as K3 does,
//               scale (bf16x2) and stmatrix A
//   MMA         warp 1 (one lane): 4 x tcgen05.mma.kind::f16 (M=128, N=BN,
//               K=16) per stage into a double-buffered fp32 TMEM accumulator;
//               tcgen05.commit frees the operand stage / publishes the tile
//   epilogue    warps 3-6: tcgen05.ld 32 lanes x 32 columns -> Y (S = 1), or
//               fp32 partials + an acq_rel ticket; the last split of a tile sums
//               the partials in split order (deterministic) and writes Y.
// The dequantised weight is rounded to bf16 once (scale * (s - z)); products
// and the K reduction run in fp32 on the tensor core.
#pragma once
#include <cuda.h>

#include "matq_common.cuh"
#include "matq_tc.cuh"

namespace mq {

struct GemmParams {
    const uint32_t* blob;
    long long step_words;  // words per (row tile, step) block
    int skip_words;        // scale words before the step's two G=128 groups (0)
    void* Y;
    int ldy;
    int B, N, K, nsteps, n_rt;
    int n_bt, n_tiles;  // token tiles, output tiles
    int S, cs;          // K splits, steps per split (of tiles t1 ..)
    int t1;             // tiles [0, t1) are whole units (full waves before a split tail)
    float* ws;          // fp32 partials [n_tiles * S][BN][128] when S > 1
    int* tickets;       // [n_tiles], zero, self-resetting
    float out_scale;
    int y_f32;
    int coop;  // S > 1 and every unit resident at once (n_tiles * S <= grid)
#ifdef MQ_GEMV_TIMING
    unsigned long long* dbg_ts;
    int dbg_slot;
#endif
};
#ifdef MQ_GEMV_TIMING
#define MQ_GTS(ev) do { if (blockIdx.x < 160) p.dbg_ts[((size_t)p.dbg_slot * 160 + blockIdx.x) * 6 + (ev)] = gtimer_gemm(); } while (0)
__device__ __forceinline__ unsigned long long gtimer_gemm() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#else
#define MQ_GTS(ev) do { } while (0)
#endif

constexpr int kGemmThreads = 23 * 32;
constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;  // K columns per operand stage (one swizzle atom)
constexpr uint32_t kGemmABytes = kGemmBM * kGemmBK * 2;  // 16 KB
// warp 0: activation-tile producer, warp 1: TMEM + MMA, warp 2: raw-weight producer,
// warps 3..6: epilogue (any 4 consecutive warps cover the 4 TMEM lane quadrants),
// warps 7..22: decoders (row tile dw & 7, word pair dw >> 3)
constexpr int kEpiWarp0 = 3, kDecWarp0 = 7, kNumDecWarps = 16, kWarpProd = 0, kWarpMma = 1, kWarpW = 2;
constexpr int kRowTiles = kGemmBM / 16;  // raw blocks per step (8)
constexpr uint32_t kSmemBudget = 227 * 1024;

__host__ __device__ constexpr uint32_t gemm_raw_block_bytes(int npl) { return 128u + 512u * (uint32_t)npl; }

template <int BN, int NPL>
struct GemmSmem {
    static constexpr uint32_t kBBytes = (uint32_t)BN * kGemmBK * 2;
    static constexpr uint32_t kOpBytes = kGemmABytes + kBBytes;
    static constexpr uint32_t kRawBytes = kRowTiles * gemm_raw_block_bytes(NPL);
    static constexpr uint32_t kFixed = 1024 + 512;  // alignment slack + barriers
    static constexpr int RS = (kFixed + 3 * kOpBytes + 3 * kRawBytes <= kSmemBudget)   ? 3
                            : (kFixed + 2 * kOpBytes + 2 * kRawBytes <= kSmemBudget) ? 2
                                                                                       : 1;
    // operand stages: as many as fit beside the raw ring, up to one step (4; 8 measured
    // neutral at B = 64-256: the decoders are not waiting on the ring depth).
    // NS >= 3 keeps a decoder from lapping another on a slot (its stages are at most
    // 3 apart); NS = 2 (BN = 512) gives each decoder warp its own slot instead
#ifndef MQ_GEMM_MAX_NS
#define MQ_GEMM_MAX_NS 4
#endif
    static constexpr int fit_ns(int n) {
        return (n <= 2 || kFixed + (uint32_t)n * kOpBytes + RS * kRawBytes <= kSmemBudget) ? n : fit_ns(n - 1);
    }
    static constexpr int NS = fit_ns(MQ_GEMM_MAX_NS);
    static constexpr uint32_t kRawOff = NS * kOpBytes;
    static constexpr uint32_t kBarOff = kRawOff + RS * kRawBytes;
    static constexpr uint32_t kBytes = kBarOff + kFixed;
    static_assert(kBytes <= kSmemBudget, "K4 shared memory budget");
};

template <int R, bool CHILD, int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmx, const GemmParams p) {
    constexpr int NPL = PlaneCount<R, CHILD>::value;
    using SM = GemmSmem<BN, NPL>;
    constexpr int NS = SM::NS, RS = SM::RS;
    // BN = 512 (two 256-token halves of one decoded weight tile): two N = 256 MMAs per
    // k16 into one 512-column accumulator, which fills TMEM, so it is single-buffered
    constexpr int kMmaN = BN > 256 ? 256 : BN, kNB = BN / kMmaN;
    constexpr int kNBuf = 2 * BN <= 512 ? 2 : 1;
    constexpr uint32_t kTmemCols = kNBuf * BN < 32 ? 32 : kNBuf * BN;
    auto tbuf = [&](int ui) { return kNBuf == 2 ? (ui & 1) : 0; };
    auto tpar = [&](int ui) { return kNBuf == 2 ? ((ui >> 1) & 1) : (ui & 1); };
    constexpr uint32_t kBlk = gemm_raw_block_bytes(NPL);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t base = (smem_addr(smem_raw) + 1023u) & ~1023u;
    auto a_st = [&](int s) { return base + (uint32_t)s * SM::kOpBytes; };
    auto b_st = [&](int s) { return base + (uint32_t)s * SM::kOpBytes + kGemmABytes; };
    auto raw_st = [&](int s) { return base + SM::kRawOff + (uint32_t)s * SM::kRawBytes; };
    const uint32_t bar0 = base + SM::kBarOff;
    auto op_full = [&](int s) { return bar0 + 8u * s; };
    auto op_empty = [&](int s) { return bar0 + 8u * (NS + s); };
    auto raw_full = [&](int s) { return bar0 + 8u * (2 * NS + s); };
    auto raw_empty = [&](int s) { return bar0 + 8u * (2 * NS + RS + s); };
    auto tfull = [&](int b) { return bar0 + 8u * (2 * NS + 2 * RS + b); };
    auto tempty = [&](int b) { return bar0 + 8u * (2 * NS + 2 * RS + 2 + b); };
    const uint32_t tmem_slot = bar0 + 8u * (2 * NS + 2 * RS + 4);
    const uint32_t flag_slot = tmem_slot + 4;
    uint8_t* const gen_base = smem_raw + (base - smem_addr(smem_raw));
    volatile uint32_t* tmem_slot_ptr = reinterpret_cast<volatile uint32_t*>(gen_base + (tmem_slot - base));
    volatile int* flag_ptr = reinterpret_cast<volatile int*>(gen_base + (flag_slot - base));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(op_full(s), 1 + kRowTiles);  // the X tile + one decoder per row tile
            mbar_init(op_empty(s), 1);
        }
        for (int s = 0; s < RS; ++s) {
            mbar_init(raw_full(s), 1);
            mbar_init(raw_empty(s), kNumDecWarps);
        }
        for (int b = 0; b < kNBuf; ++b) {
            mbar_init(tfull(b), 1);
            mbar_init(tempty(b), 4);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmx);
    }
    if (warp == kWarpMma) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot_ptr;
    pdl_launch_dependents();
    if (threadIdx.x == 0) MQ_GTS(0);

    const int n_units = p.t1 + (p.n_tiles - p.t1) * p.S;
    const int my_units = (int)blockIdx.x < n_units ? (n_units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    // unit -> (tile, split, step range); units [0, t1) are whole tiles, then consecutive
    // units are the S splits of one tile
    auto unit_of = [&](int ui, int& tile, int& split, int& st0, int& nst) {
        const int u = (int)blockIdx.x + ui * (int)gridDim.x;
        if (u < p.t1) {
            tile = u;
            split = 0;
            st0 = 0;
            nst = p.nsteps;
            return;
        }
        const int v = u - p.t1;
        tile = p.t1 + v / p.S;
        split = v - (tile - p.t1) * p.S;
        st0 = split * p.cs;
        nst = max(0, min(p.nsteps, st0 + p.cs) - st0);
    };
    auto is_split = [&](int tile) { return p.S > 1 && tile >= p.t1; };
    // fp32 partials of the split tiles: [(tile - t1) * S + split][BN / 4][128][4]
    auto part_base = [&](int tile) { return p.ws + (long long)(tile - p.t1) * p.S * (BN * kGemmBM); };

    // flattened (unit, step) sequence of this CTA
    int total_steps = 0;
    for (int ui = 0; ui < my_units; ++ui) {
        int tile, split, st0, nst;
        unit_of(ui, tile, split, st0, nst);
        total_steps += nst;
    }

    if (warp == kWarpProd) {
        // ---------------- producer: activation tiles ----------------------------
        if (lane == 0) {
            pdl_wait();  // X is written by the previous kernel
            int ks = 0;
            for (int ui = 0; ui < my_units; ++ui) {
                int tile, split, st0, nst;
                unit_of(ui, tile, split, st0, nst);
                const int bt = tile % p.n_bt;
                for (int si = 0; si < nst; ++si) {
                    for (int kk = 0; kk < 4; ++kk, ++ks) {
                        const int s = ks % NS;
                        mbar_wait(op_empty(s), ((ks / NS) & 1) ^ 1);
                        mbar_expect_tx(op_full(s), SM::kBBytes);
#pragma unroll
                        for (int nb = 0; nb < kNB; ++nb)
                            tma_load_2d(b_st(s) + (uint32_t)(nb * kMmaN * 128), &tmx, (st0 + si) * 256 + kk * kGemmBK,
                                        bt * BN + nb * kMmaN, op_full(s));
                    }
                }
            }
        }
        __syncwarp();  // lane 0's role loop rejoins its warp before the final barrier
    } else if (warp == kWarpW) {
        // ---------------- producer: raw weight blocks (independent of X: no PDL wait) --
        if (lane == 0) {
            int r_ui = 0, r_si = 0;
            for (int r_f = 0; r_f < total_steps; ++r_f) {
                int tile, split, st0, nst;
                unit_of(r_ui, tile, split, st0, nst);
                const int rt0 = (tile / p.n_bt) * kRowTiles;
                const int nvalid = min(kRowTiles, p.n_rt - rt0);
                const int s = r_f % RS;
                mbar_wait(raw_empty(s), ((r_f / RS) & 1) ^ 1);
                mbar_expect_tx(raw_full(s), (uint32_t)nvalid * kBlk);
                const int st = st0 + r_si;
                for (int d = 0; d < nvalid; ++d)
                    bulk_g2s_nohint(raw_st(s) + (uint32_t)d * kBlk,
                                    p.blob + ((long long)(rt0 + d) * p.nsteps + st) * p.step_words + p.skip_words,
                                    kBlk, raw_full(s));
                if (++r_si == nst) {
                    r_si = 0;
                    ++r_ui;
                }
            }
        }
        __syncwarp();  // lane 0's role loop rejoins its warp before the final barrier
    } else if (warp == kWarpMma) {
        // ---------------- MMA issuer ----------------------------------------
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(kGemmBM, kMmaN);
            int ks = 0;
            for (int ui = 0; ui < my_units; ++ui) {
                int tile, split, st0, nst;
                unit_of(ui, tile, split, st0, nst);
                const int buf = tbuf(ui);
                mbar_wait(tempty(buf), tpar(ui) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + (uint32_t)(buf * BN);
                for (int kk = 0; kk < 4 * nst; ++kk, ++ks) {
                    const int s = ks % NS;
                    mbar_wait(op_full(s), (ks / NS) & 1);
                    if (ks == 0) MQ_GTS(2);
                    tc_fence_after();
#pragma unroll
                    for (int k16 = 0; k16 < kGemmBK / 16; ++k16) {
                        const uint64_t ad = umma_desc_k_sw128(a_st(s) + (uint32_t)k16 * 32u);
#pragma unroll
                        for (int nb = 0; nb < kNB; ++nb) {
                            const uint64_t bd =
                                umma_desc_k_sw128(b_st(s) + (uint32_t)(nb * kMmaN * 128) + (uint32_t)k16 * 32u);
                            umma_bf16(d + (uint32_t)(nb * kMmaN), ad, bd, idesc, (kk | k16) != 0);
                        }
                    }
                    umma_commit(op_empty(s));
                }
                umma_commit(tfull(buf));
            }
            MQ_GTS(3);
        }
        __syncwarp();  // lane 0's role loop rejoins its warp before the final barrier
    } else if (warp >= kEpiWarp0) {
        // ---------------- epilogue: TMEM -> Y / split-K partials ---------------------
        auto epilogue = [&](int ui) {
            const int q = warp & 3;                  // TMEM lane quadrant of this warp
            const int et = 32 * q + lane;            // 0..127 = TMEM lane = tile row
            int tile, split, st0, nst;
            unit_of(ui, tile, split, st0, nst);
            const int mt = tile / p.n_bt, bt = tile % p.n_bt;
            const int buf = tbuf(ui);
            mbar_wait(tfull(buf), tpar(ui));
            if (warp == kEpiWarp0 && lane == 0 && ui == my_units - 1) MQ_GTS(4);
            tc_fence_after();
            const int row = mt * kGemmBM + et;
            const int b_lim = min(BN, p.B - bt * BN);
            auto store_y = [&](int j, float v) {
                const long long o = (long long)(bt * BN + j) * p.ldy + row;
                if (p.y_f32) reinterpret_cast<float*>(p.Y)[o] = v;
                else reinterpret_cast<uint16_t*>(p.Y)[o] = f32_to_bf16_rn(v);
            };
            // split-K partial of this unit: [BN / 4][128 rows][4] floats (float4 per row and
            // 4 columns: the TMEM lane's 32 columns go out as 8 vector stores)
            const bool split_tile = is_split(tile);
            float4* part4 = split_tile ? reinterpret_cast<float4*>(part_base(tile) + (long long)split * (BN * kGemmBM))
                                       : nullptr;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * BN + 32 * c), v);
                tmem_ld_wait();
                if (!split_tile) {
                    if (row < p.N) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (32 * c + j < b_lim) store_y(32 * c + j, __uint_as_float(v[j]));
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        part4[(8 * c + i) * kGemmBM + et] =
                            make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                        __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                }
            }
            // TMEM buffer can be refilled as soon as it is read
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty(buf));
            if (split_tile) {
                // publish the partial.  coop (every unit resident at once): the whole CTA
                // reduces a 1/S share of the tile's columns after the role loops (below);
                // otherwise the last split to arrive reduces the tile here.  Split order
                // either way (deterministic).
                __threadfence();
                named_bar_sync(1, 128);
                if (et == 0) *flag_ptr = atom_add_acq_rel(p.tickets + tile, 1);
                named_bar_sync(1, 128);
                if (p.coop) return;
                const int arrived = *flag_ptr;
                const int q_hi = arrived == p.S - 1 ? (b_lim + 3) >> 2 : 0;  // column quads reduced here
                __threadfence();
                const float4* t0 = reinterpret_cast<const float4*>(part_base(tile));
                const long long sstride = (long long)(BN / 4) * kGemmBM;  // float4s per split
                if (row < p.N) {
#pragma unroll 1
                    for (int q0 = 0; q0 < q_hi; q0 += 4) {
                        float4 acc[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                        for (int sp = 0; sp < p.S; ++sp) {  // split order: deterministic
                            float4 v[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                v[u] = q0 + u < q_hi ? __ldcg(t0 + sp * sstride + (long long)(q0 + u) * kGemmBM + et)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                acc[u].x += v[u].x; acc[u].y += v[u].y; acc[u].z += v[u].z; acc[u].w += v[u].w;
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int j = 4 * (q0 + u);
                            if (q0 + u < q_hi) {
                                if (j < b_lim) store_y(j, acc[u].x);
                                if (j + 1 < b_lim) store_y(j + 1, acc[u].y);
                                if (j + 2 < b_lim) store_y(j + 2, acc[u].z);
                                if (j + 3 < b_lim) store_y(j + 3, acc[u].w);
                            }
                        }
                    }
                }
                named_bar_sync(1, 128);
                if (et == 0 && arrived == p.S - 1) p.tickets[tile] = 0;
                named_bar_sync(1, 128);  // flag slot reuse
            }
        };
        if (warp < kDecWarp0) {
            for (int ui = 0; ui < my_units; ++ui) epilogue(ui);
        } else {
            // ---------------- decoders: raw blocks -> bf16 A operand -----------------
            const int dw = warp - kDecWarp0;
            const int rtl = dw & (kRowTiles - 1), half = dw >> 3;  // row tile, word pair
            // with only 2 operand stages (BN = 512) the two decoders of a row tile must not
            // share a stage slot (a warp could lap the other by a whole mbarrier phase, which
            // the parity wait cannot see): decoder `half` takes words {half, half + 2}, both
            // in slot `half`; otherwise words {2 half, 2 half + 1}
            constexpr bool kSlotPairs = NS == 2;
            auto word_of = [&](int wi) { return kSlotPairs ? half + 2 * wi : 2 * half + wi; };
            const int g = lane >> 2;
            // stmatrix row address: matrix j = lane >> 3 holds rows +8 (j & 1), columns +8 (j >> 1)
            const int jm = lane >> 3;
            const uint32_t row_off = (uint32_t)(16 * rtl + (lane & 7) + 8 * (jm & 1)) * 128u;
            const uint32_t swz = (uint32_t)(lane & 7);
            int fglob = 0;
            for (int ui = 0; ui < my_units; ++ui) {
                int tile, split, st0, nst;
                unit_of(ui, tile, split, st0, nst);
                const bool valid = (tile / p.n_bt) * kRowTiles + rtl < p.n_rt;
#pragma unroll 1
                for (int f = 0; f < nst; ++f, ++fglob) {
                    const int rsl = fglob % RS;
                    mbar_wait(raw_full(rsl), (fglob / RS) & 1);
                    if (fglob == 0 && dw == 0 && lane == 0) MQ_GTS(1);
                    uint2 raw[NPL];  // the two words (of four) of this decoder's word pair
                    uint32_t s_lo[2], s_hi[2];  // per word of the pair: group scale, rows g / g + 8
                    const uint32_t blk = raw_st(rsl) + (uint32_t)rtl * kBlk;
                    if (valid) {
#pragma unroll
                        for (int wi = 0; wi < 2; ++wi) {
                            const int grp = word_of(wi) >> 1;  // 128-column scale group of the word
                            s_lo[wi] = bf16x2_splat(lds32f(blk + 4u * (16 * grp + g)) * p.out_scale);
                            s_hi[wi] = bf16x2_splat(lds32f(blk + 4u * (16 * grp + g + 8)) * p.out_scale);
                        }
                        if constexpr (kSlotPairs) {
#pragma unroll
                            for (int jj = 0; jj < NPL; ++jj) {
                                const uint32_t wb = blk + 128u + 512u * jj + 16u * lane;
                                raw[jj] = make_uint2(__float_as_uint(lds32f(wb + 4u * word_of(0))),
                                                     __float_as_uint(lds32f(wb + 4u * word_of(1))));
                            }
                        } else {
#pragma unroll
                            for (int jj = 0; jj < NPL; ++jj)
                                raw[jj] = lds64(blk + 128u + 512u * jj + 16u * lane + 8u * half);
                        }
                    } else {
                        s_lo[0] = s_lo[1] = s_hi[0] = s_hi[1] = 0u;
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(raw_empty(rsl));
#ifndef MQ_GEMM_PREDECODE
#define MQ_GEMM_PREDECODE 1
#endif
                    if (MQ_GEMM_PREDECODE) {
                        // decode both words of the pair before waiting for their operand
                        // stages: two independent dependency chains in flight, and the
                        // decode overlaps the MMA still reading those stages
                        uint32_t A2[2][16];
                        if (valid) {
#pragma unroll
                            for (int wi = 0; wi < 2; ++wi) {
                                uint32_t T[NPL];
#pragma unroll
                                for (int jj = 0; jj < NPL; ++jj) T[jj] = wi ? raw[jj].y : raw[jj].x;
                                uint32_t Sl[R];
                                slice_loaded<R, CHILD>(T, Sl);
                                decode_word<R, false>(Sl, A2[wi]);
#pragma unroll
                                for (int qq = 0; qq < 16; ++qq)
                                    A2[wi][qq] = hmul2_bf16(A2[wi][qq], (qq & 1) ? s_hi[wi] : s_lo[wi]);
                            }
                        }
#pragma unroll
                        for (int wi = 0; wi < 2; ++wi) {
                            const int ks = 4 * fglob + word_of(wi);
                            const int s = ks % NS;
                            mbar_wait(op_empty(s), ((ks / NS) & 1) ^ 1);
                            if (valid) {
                                const uint32_t abase = a_st(s) + row_off;
#pragma unroll
                                for (int k16 = 0; k16 < 4; ++k16) {
                                    const uint32_t chunk = (uint32_t)(2 * k16 + (jm >> 1));
                                    stmatrix_x4(abase + ((chunk ^ swz) << 4), A2[wi][4 * k16], A2[wi][4 * k16 + 1],
                                                A2[wi][4 * k16 + 2], A2[wi][4 * k16 + 3]);
                                }
                                fence_proxy_async_smem();
                            }
                            __syncwarp();
                            if (lane == 0) mbar_arrive(op_full(s));
                        }
                        continue;
                    }
#pragma unroll
                    for (int wi = 0; wi < 2; ++wi) {
                        const int ks = 4 * fglob + word_of(wi);
                        const int s = ks % NS;
                        mbar_wait(op_empty(s), ((ks / NS) & 1) ^ 1);
                        if (valid) {
                            uint32_t T[NPL];
#pragma unroll
                            for (int jj = 0; jj < NPL; ++jj) T[jj] = wi ? raw[jj].y : raw[jj].x;
                            uint32_t Sl[R];
                            slice_loaded<R, CHILD>(T, Sl);
                            uint32_t A[16];
                            decode_word<R, false>(Sl, A);
#pragma unroll
                            for (int qq = 0; qq < 16; ++qq) A[qq] = hmul2_bf16(A[qq], (qq & 1) ? s_hi[wi] : s_lo[wi]);
                            const uint32_t abase = a_st(s) + row_off;
#pragma unroll
                            for (int k16 = 0; k16 < 4; ++k16) {
                                const uint32_t chunk = (uint32_t)(2 * k16 + (jm >> 1));
                                stmatrix_x4(abase + ((chunk ^ swz) << 4), A[4 * k16], A[4 * k16 + 1],
                                            A[4 * k16 + 2], A[4 * k16 + 3]);
                            }
                            fence_proxy_async_smem();
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive(op_full(s));
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    int l_tile = 0, l_split = 0, l_st0 = 0, l_nst = 0;
    if (my_units > 0) unit_of(my_units - 1, l_tile, l_split, l_st0, l_nst);
    if (p.coop && my_units > 0 && is_split(l_tile)) {
        // coop split-K: once all S partials of this CTA's (last, split) tile exist, all 23
        // warps reduce this split's 1/S share of the columns (flattened (column quad, row)
        // tasks, rows fastest: coalesced loads and Y stores; four tasks in flight per thread)
        const int tile = l_tile, split = l_split;
        const int mt = tile / p.n_bt, bt = tile % p.n_bt;
        const int b_lim = min(BN, p.B - bt * BN);
        const int nq = (b_lim + 3) >> 2;
        const int q_lo = split * nq / p.S, q_hi = (split + 1) * nq / p.S;
        if (threadIdx.x == 0)
            while (ld_acquire_s32(p.tickets + tile) < p.S) {
            }
        __syncthreads();
        __threadfence();
        const float4* t0 = reinterpret_cast<const float4*>(part_base(tile));
        const long long sstride = (long long)(BN / 4) * kGemmBM;
        const int ntask = (q_hi - q_lo) * kGemmBM;
        constexpr int kU = 4;
#pragma unroll 1
        for (int base = threadIdx.x; base < ntask; base += kU * kGemmThreads) {
            float4 acc[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int sp = 0; sp < p.S; ++sp) {
                float4 v[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const int task = base + u * kGemmThreads;
                    v[u] = task < ntask ? __ldcg(t0 + sp * sstride + (long long)(q_lo * kGemmBM + task))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    acc[u].x += v[u].x; acc[u].y += v[u].y; acc[u].z += v[u].z; acc[u].w += v[u].w;
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int task = base + u * kGemmThreads;
                if (task >= ntask) break;
                const int q = q_lo + task / kGemmBM, et = task % kGemmBM;
                const int row = mt * kGemmBM + et;
                if (row >= p.N) continue;
                const float vals[4] = {acc[u].x, acc[u].y, acc[u].z, acc[u].w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int j = 4 * q + c;
                    if (j < b_lim) {
                        const long long o = (long long)(bt * BN + j) * p.ldy + row;
                        if (p.y_f32) reinterpret_cast<float*>(p.Y)[o] = vals[c];
                        else reinterpret_cast<uint16_t*>(p.Y)[o] = f32_to_bf16_rn(vals[c]);
                    }
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && atom_add_acq_rel(p.tickets + tile, 1) == 2 * p.S - 1)
            p.tickets[tile] = 0;  // the last split through resets the ticket (2 S arrivals)
    }
    if (warp == kWarpMma) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem_base);
        if (lane == 0) MQ_GTS(5);  // every warp (incl. the split-K reduction) is done
    }
}

}  // namespace mq
