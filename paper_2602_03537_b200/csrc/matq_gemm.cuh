// matq_gemm.cuh -- K4: prefill dequant-GEMM on the 5th-generation tensor cores.
//
// Y[b, n] = sum_k X[b, k] * scale[n, k / 128] * out_scale * (s_r(q[n, k]) - 2^(r-1))
// for token counts past the GEMV range (B > 32; BASELINE config C4).  The
// reference has no batched GPU path; its CPU analogue is nq_gemm
// (packed_kernels.c:177-210, driven in chunks of 16 rows by
// kernels/_core.pyx:53-63).
//
// One persistent CTA per SM, 16 warps, output tiles of 128 weight rows x BN
// tokens, K consumed 128 columns (one scale group) per pipeline stage:
//   warp 0      TMA producer: X tile [BN tokens][128 k] bf16, two 64-column
//               SWIZZLE_128B boxes per stage (tensor map, zero fill past B / K)
//   warp 1      TMEM allocator + MMA issuer: 8 x tcgen05.mma.kind::f16
//               (M=128, N=BN, K=16) per stage into a double-buffered fp32
//               accumulator in TMEM; tcgen05.commit frees the stage
//   warps 4-7   epilogue: tcgen05.ld 32 lanes x 32 columns, bf16/fp32 store
//   warps 8-15  decode producers, one 16-row tile each: stream the P8 blob
//               (r+1 planes + group scales) straight from HBM, slice + decode
//               bitsliced exactly as K3 does, multiply by the group scale
//               (bf16x2), and stmatrix the mma-fragment-ordered registers into
//               the K-major SWIZZLE_128B A operand.
// The dequantised weight is rounded to bf16 once (scale * (s - z)); the
// products and the K reduction run in fp32 on the tensor core.
#pragma once
#include <cuda.h>

#include "matq_common.cuh"
#include "matq_tc.cuh"

namespace mq {

struct GemmParams {
    const uint32_t* blob;
    long long step_words;  // words per (row tile, step) block
    int sb_words;          // scale-block words at the head of a block (32 for G = 128)
    void* Y;
    int ldy;
    int B, N, K, nsteps, n_rt;
    int n_bt, n_tiles;  // token tiles, output tiles
    float out_scale;
    int y_f32;
};

constexpr int kGemmThreads = 512;
constexpr int kGemmBM = 128;
constexpr int kGemmBK = 128;
constexpr uint32_t kGemmABytes = kGemmBM * kGemmBK * 2;  // 32 KB
constexpr int kDecWarp0 = 8, kNumDecWarps = 8, kEpiWarp0 = 4;

template <int BN>
struct GemmSmem {
    static constexpr int NS = BN <= 64 ? 4 : 3;
    static constexpr uint32_t kBBytes = (uint32_t)BN * kGemmBK * 2;
    static constexpr uint32_t kBarOff = NS * (kGemmABytes + kBBytes);
    static constexpr uint32_t kBytes = kBarOff + 256 + 1024;  // + barriers, + alignment slack
};

template <int R, bool CHILD, int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmx, const GemmParams p) {
    constexpr int NPL = PlaneCount<R, CHILD>::value;
    using SM = GemmSmem<BN>;
    constexpr int NS = SM::NS;
    constexpr uint32_t kTmemCols = 2 * BN;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t base = (smem_addr(smem_raw) + 1023u) & ~1023u;
    auto a_st = [&](int s) { return base + (uint32_t)s * kGemmABytes; };
    auto b_st = [&](int s) { return base + NS * kGemmABytes + (uint32_t)s * SM::kBBytes; };
    const uint32_t bar0 = base + SM::kBarOff;
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (NS + s); };
    auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * NS + b); };
    auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * NS + 2 + b); };
    const uint32_t tmem_slot = bar0 + 8u * (2 * NS + 4);
    uint32_t* tmem_slot_ptr =
        reinterpret_cast<uint32_t*>(smem_raw + (tmem_slot - smem_addr(smem_raw)));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(full_bar(s), 1 + kNumDecWarps);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b), 4);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmx);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot_ptr;
    pdl_launch_dependents();

    const int nst = p.nsteps;
    const int my_tiles = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (warp == 0) {
        // ---------------- TMA producer: activations -------------------------
        if (lane == 0) {
            pdl_wait();  // X is written by the previous kernel
            int ks = 0;
            for (int ti = 0; ti < my_tiles; ++ti) {
                const int tile = blockIdx.x + ti * gridDim.x;
                const int bt = tile % p.n_bt;
                for (int kk = 0; kk < 2 * nst; ++kk, ++ks) {
                    const int s = ks % NS;
                    mbar_wait(empty_bar(s), ((ks / NS) & 1) ^ 1);
                    mbar_expect_tx(full_bar(s), SM::kBBytes);
                    const int k0 = kk * kGemmBK;
                    tma_load_2d(b_st(s), &tmx, k0, bt * BN, full_bar(s));
                    tma_load_2d(b_st(s) + BN * 128, &tmx, k0 + 64, bt * BN, full_bar(s));
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------------------------------
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(kGemmBM, BN);
            int ks = 0;
            for (int ti = 0; ti < my_tiles; ++ti) {
                const int buf = ti & 1;
                mbar_wait(tempty_bar(buf), ((ti >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + (uint32_t)(buf * BN);
                for (int kk = 0; kk < 2 * nst; ++kk, ++ks) {
                    const int s = ks % NS;
                    mbar_wait(full_bar(s), (ks / NS) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int k16 = 0; k16 < kGemmBK / 16; ++k16) {
                        const uint32_t atom = (uint32_t)(k16 >> 2), off = (uint32_t)(k16 & 3) * 32u;
                        const uint64_t ad = umma_desc_k_sw128(a_st(s) + atom * 16384u + off);
                        const uint64_t bd = umma_desc_k_sw128(b_st(s) + atom * (BN * 128u) + off);
                        umma_bf16(d, ad, bd, idesc, (kk | k16) != 0);
                    }
                    umma_commit(empty_bar(s));
                }
                umma_commit(tfull_bar(buf));
            }
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        // ---------------- epilogue: TMEM -> Y ----------------------------------
        const int q = warp & 3;
        for (int ti = 0; ti < my_tiles; ++ti) {
            const int tile = blockIdx.x + ti * gridDim.x;
            const int mt = tile / p.n_bt, bt = tile % p.n_bt;
            const int buf = ti & 1;
            mbar_wait(tfull_bar(buf), (ti >> 1) & 1);
            tc_fence_after();
            const int row = mt * kGemmBM + 32 * q + lane;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * BN + 32 * c), v);
                tmem_ld_wait();
                if (row < p.N) {
                    const int b0 = bt * BN + 32 * c;
                    if (p.y_f32) {
                        float* Y = reinterpret_cast<float*>(p.Y);
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (b0 + j < p.B) Y[(long long)(b0 + j) * p.ldy + row] = __uint_as_float(v[j]);
                    } else {
                        uint16_t* Y = reinterpret_cast<uint16_t*>(p.Y);
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (b0 + j < p.B)
                                Y[(long long)(b0 + j) * p.ldy + row] = f32_to_bf16_rn(__uint_as_float(v[j]));
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar(buf));
        }
    } else if (warp >= kDecWarp0) {
        // ---------------- decode producers: P8 blob -> bf16 A operand -----------
        const int dw = warp - kDecWarp0;
        const int g = lane >> 2;
        const int total = my_tiles * nst;
        // stmatrix row address: matrix j = lane >> 3 holds rows +8 (j & 1), columns +8 (j >> 1)
        const int j = lane >> 3;
        const uint32_t row_off = (uint32_t)(16 * dw + (lane & 7) + 8 * (j & 1)) * 128u;
        const uint32_t swz = (uint32_t)(lane & 7);
        auto block_of = [&](int f) -> const uint32_t* {
            const int tile = blockIdx.x + (f / nst) * gridDim.x;
            const int st = f - (f / nst) * nst;
            const int rt = (tile / p.n_bt) * (kGemmBM / 16) + dw;
            return rt < p.n_rt ? p.blob + ((long long)rt * nst + st) * p.step_words : nullptr;
        };
        uint4 raw[NPL], nxt[NPL];
        float sc[4], nsc[4];
        auto load = [&](const uint32_t* b, uint4 (&rw)[NPL], float (&s4)[4]) {
            if (b == nullptr) return;
            s4[0] = ldg_f32(reinterpret_cast<const float*>(b) + g);
            s4[1] = ldg_f32(reinterpret_cast<const float*>(b) + g + 8);
            s4[2] = ldg_f32(reinterpret_cast<const float*>(b) + 16 + g);
            s4[3] = ldg_f32(reinterpret_cast<const float*>(b) + 24 + g);
#pragma unroll
            for (int jj = 0; jj < NPL; ++jj)
                rw[jj] = ldg_stream(reinterpret_cast<const uint4*>(b + p.sb_words + jj * 128) + lane);
        };
        const uint32_t* cur = total > 0 ? block_of(0) : nullptr;
        load(cur, raw, sc);
#pragma unroll 1
        for (int f = 0; f < total; ++f) {
            const uint32_t* nb = f + 1 < total ? block_of(f + 1) : nullptr;
            load(nb, nxt, nsc);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ks = 2 * f + h;
                const int s = ks % NS;
                mbar_wait(empty_bar(s), ((ks / NS) & 1) ^ 1);
                if (cur != nullptr) {
                    const uint32_t s_lo = bf16x2_splat(sc[2 * h] * p.out_scale);
                    const uint32_t s_hi = bf16x2_splat(sc[2 * h + 1] * p.out_scale);
                    const uint32_t abase = a_st(s) + row_off;
#pragma unroll
                    for (int wi = 0; wi < 2; ++wi) {
                        const int w = 2 * h + wi;
                        uint32_t T[NPL];
#pragma unroll
                        for (int jj = 0; jj < NPL; ++jj) T[jj] = word_of(raw[jj], w);
                        uint32_t Sl[R];
                        slice_loaded<R, CHILD>(T, Sl);
                        uint32_t A[16];
                        decode_word<R, false>(Sl, A);
#pragma unroll
                        for (int qq = 0; qq < 16; ++qq) A[qq] = hmul2_bf16(A[qq], (qq & 1) ? s_hi : s_lo);
#pragma unroll
                        for (int k16 = 0; k16 < 4; ++k16) {
                            const uint32_t chunk = (uint32_t)(2 * k16 + (j >> 1));
                            stmatrix_x4(abase + (uint32_t)wi * 16384u + ((chunk ^ swz) << 4), A[4 * k16],
                                        A[4 * k16 + 1], A[4 * k16 + 2], A[4 * k16 + 3]);
                        }
                    }
                    fence_proxy_async_smem();
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(full_bar(s));
            }
            cur = nb;
#pragma unroll
            for (int jj = 0; jj < NPL; ++jj) raw[jj] = nxt[jj];
#pragma unroll
            for (int i = 0; i < 4; ++i) sc[i] = nsc[i];
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem_base);
    }
}

}  // namespace mq
