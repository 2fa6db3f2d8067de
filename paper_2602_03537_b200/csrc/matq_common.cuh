// matq_common.cuh -- device building blocks shared by every matq kernel.
//
// Device parent layout "P8":
//   planes : uint32[8][Np/16][Kp/256][32 lanes][4 words]   plane 0 = code MSB
//   tscales: fp32 [Np/16][ngp][16]                          tiled group scales
// Np = N rounded up to 16, Kp = K rounded up to 256, ngp = ceil(Kp / G).
// One uint32 word of one plane holds one bit of 32 weights of a 16-row x
// 64-column block, arranged so that the word a lane loads is exactly the set
// of weights that lane holds in the A fragments of four mma.m16n8k16 steps:
//   lane = 4g + t, bit p in [0,16) and p + 16 of word w of a 256-column step:
//     s = p >> 2 (k16 step), q = p & 3 (A register a0..a3)
//     row = 16*rt + g + 8*(q & 1)
//     col = 256*step + 64*w + 16*s + 8*(q >> 1) + 2*t + (bit >= 16)
// so a warp's 128-bit load of one plane is 512 contiguous bytes, and every
// r-slice reads planes 0..r (r+1 planes, all 8 at r = 8) and nothing else.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define MQ_HD __host__ __device__ __forceinline__

namespace mq {

constexpr int kTileRows = 16;   // rows per warp tile (mma M)
constexpr int kStepCols = 256;  // columns per 128-bit load per plane
constexpr int kWordCols = 64;   // columns per lane word

__host__ __device__ constexpr int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }
__host__ __device__ constexpr int pad16(int n) { return cdiv(n, 16) * 16; }
__host__ __device__ constexpr int pad256(int k) { return cdiv(k, 256) * 256; }

// Position of bit `bit` (0..31) of word `w` (0..3) for lane `lane` within a
// (row tile, step) block: returns (row offset in tile, column offset in step).
__host__ __device__ __forceinline__ void word_bit_pos(int lane, int w, int bit, int& row, int& col) {
    const int g = lane >> 2, t = lane & 3;
    const int p = bit & 15, h = bit >> 4;
    const int s = p >> 2, q = p & 3;
    row = g + 8 * (q & 1);
    col = 64 * w + 16 * s + 8 * (q >> 1) + 2 * t + h;
}

// Step-interleaved blob layout.  For every (row tile, step):
//   [scale block: spg groups x 16 rows fp32][plane 0 slab]...[plane P-1 slab]
// with one slab = 32 lanes x 4 words.  A slice-r GEMV step reads the first
// scale_words + (r+1) slabs -- one contiguous bulk copy.  spg = 256/G for
// G in {32, 64, 128}, 1 when G is a multiple of 256 (the step's group), and
// 0 for other group sizes (then a separate tiled scale array [Np/16][ngp][16]
// is used).
struct Layout {
    int N, K, Np, Kp, n_rt, nsteps, nplanes, G, spg, ngp;
    long long step_words;  // words per (row tile, step) block
    __host__ __device__ static Layout make(int N, int K, int G, int nplanes) {
        Layout L{};
        L.N = N; L.K = K; L.G = G; L.nplanes = nplanes;
        L.Np = pad16(N); L.Kp = pad256(K);
        L.n_rt = L.Np / 16; L.nsteps = L.Kp / 256;
        L.spg = (G > 0 && 256 % G == 0 && G % 32 == 0) ? 256 / G : ((G > 0 && G % 256 == 0) ? 1 : 0);
        L.ngp = G > 0 ? cdiv(L.Kp, G) : 0;
        L.step_words = 16LL * L.spg + 128LL * nplanes;
        return L;
    }
    __host__ __device__ long long total_words() const { return (long long)n_rt * nsteps * step_words; }
    __host__ __device__ long long block(int rt, int st) const {
        return ((long long)rt * nsteps + st) * step_words;
    }
    __host__ __device__ long long plane_word(int rt, int st, int plane, int lane, int w) const {
        return block(rt, st) + 16LL * spg + 128LL * plane + lane * 4 + w;
    }
    // scale of (row-in-tile r16, column col) inside the step's scale block
    __host__ __device__ long long scale_word(int rt, int st, int r16, int col_in_step) const {
        const int gi = spg > 1 ? col_in_step / G : 0;
        return block(rt, st) + gi * 16 + r16;
    }
};

// ----------------------------------------------------------------------------
// bf16 constants (exact small dyadic values), computed at compile time.
__host__ __device__ constexpr uint32_t bf16_bits(int num, int sh) {  // num * 2^-sh
    if (num == 0) return 0u;
    uint32_t sgn = num < 0 ? 0x8000u : 0u;
    int a = num < 0 ? -num : num;
    int e = 0;
    while ((a >> e) > 1) ++e;
    uint32_t m = e <= 7 ? (((uint32_t)a << (7 - e)) & 0x7Fu) : (((uint32_t)a >> (e - 7)) & 0x7Fu);
    return sgn | ((uint32_t)(e - sh + 127) << 7) | m;
}
__host__ __device__ constexpr uint32_t x2(uint32_t h) { return h | (h << 16); }
static_assert(bf16_bits(128, 0) == 0x4300u, "bf16 128");
static_assert(bf16_bits(-130, 0) == 0xC302u, "bf16 -130");
static_assert(bf16_bits(1, 4) == 0x3D80u, "bf16 1/16");

// Host emulation (tests/test_layout_emulation.py): every use below produces an
// exactly representable small integer, so float arithmetic + truncation to
// bf16 reproduces the device instruction bit for bit.
MQ_HD float host_bf16(uint32_t h) {
    union { uint32_t u; float f; } v;
    v.u = (h & 0xFFFFu) << 16;
    return v.f;
}
MQ_HD uint32_t host_to_bf16(float f) {
    union { uint32_t u; float f; } v;
    v.f = f;
    return v.u >> 16;
}
MQ_HD uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
#ifdef __CUDA_ARCH__
    uint32_t d;
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
#else
    const float lo = host_bf16(a) * host_bf16(b) + host_bf16(c);
    const float hi = host_bf16(a >> 16) * host_bf16(b >> 16) + host_bf16(c >> 16);
    return host_to_bf16(lo) | (host_to_bf16(hi) << 16);
#endif
}
MQ_HD uint32_t hsub2(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    uint32_t d;
    asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
#else
    const float lo = host_bf16(a) - host_bf16(b);
    const float hi = host_bf16(a >> 16) - host_bf16(b >> 16);
    return host_to_bf16(lo) | (host_to_bf16(hi) << 16);
#endif
}

// ----------------------------------------------------------------------------
// Pipe-balanced integer primitives.  The decode is ALU-bound, and the SM has
// two half-rate integer-capable pipes: LOP3/SHF issue on the ALU pipe,
// IMAD/HFMA2 on the FMA pipe.  Left shifts are written as IMAD.SHL and right
// shifts as IMAD.HI (x * 2^(32-s) >> 32) so they land on the FMA pipe, and
// every 3-input boolean is one explicit LOP3 (ptxas otherwise splits
// (x & imm) | imm into two).
template <uint32_t LUT>
MQ_HD uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
#ifdef __CUDA_ARCH__
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
#else
    uint32_t d = 0;
    for (int i = 0; i < 8; ++i)
        if ((LUT >> i) & 1u)
            d |= ((i & 4) ? a : ~a) & ((i & 2) ? b : ~b) & ((i & 1) ? c : ~c);
    return d;
#endif
}
// LUTs over (a = 0xF0, b = 0xCC, c = 0xAA)
constexpr uint32_t kAndOr = 0xEA;   // (a & b) | c
constexpr uint32_t kAndXor = 0x6A;  // (a & b) ^ c
constexpr uint32_t kSelect = 0xE4;  // (a & c) | (b & ~c)

template <int S>
MQ_HD uint32_t shl(uint32_t x) {
#ifdef __CUDA_ARCH__
    uint32_t d;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "n"(1u << S));
    return d;
#else
    return x << S;
#endif
}
// Right shifts.  Measured on B200 (scripts/micro/op_rate.cu): LOP3, SHF, PRMT
// and HFMA2 retire 2 warp-instr/cycle/SM, IMAD.HI only 1.  MQ_SHR_MODE picks
// the implementation for the network (shr) and field extraction (shr_x):
// 0 = all IMAD.HI, 1 = all SHF, 2 = IMAD.HI in the network + SHF/PRMT in extraction.
#ifndef MQ_SHR_MODE
#define MQ_SHR_MODE 1
#endif
template <int S, bool IMAD>
MQ_HD uint32_t shr_impl(uint32_t x) {
    static_assert(S > 0 && S < 32, "shift");
#ifdef __CUDA_ARCH__
    uint32_t d;
    if constexpr (IMAD) {
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "n"(1u << (32 - S)));
    } else if constexpr (S == 8) {
        asm("prmt.b32 %0, %1, 0, 0x4321;" : "=r"(d) : "r"(x));  // bytes >> 8, zero-fill
    } else {
        asm("shr.b32 %0, %1, %2;" : "=r"(d) : "r"(x), "n"(S));
    }
    return d;
#else
    return x >> S;
#endif
}
template <int S>
MQ_HD uint32_t shr(uint32_t x) { return shr_impl<S, MQ_SHR_MODE != 1>(x); }
template <int S>
MQ_HD uint32_t shr_x(uint32_t x) { return shr_impl<S, MQ_SHR_MODE == 0>(x); }

// Field of R bits at bit offset O of both 16-bit halves of w -> bf16x2 of
// (field - 2^(R-1)), exact.  (w & mask) | 0x4300 is bf16 128 + field*2^O; one
// bf16x2 FMA by 2^-O with addend -(128*2^-O + z) lands on field - z exactly.
template <int R, int O>
MQ_HD uint32_t field_bf16(uint32_t w) {
    static_assert(O + R <= 7, "field must sit inside the bf16 mantissa");
    constexpr uint32_t m = ((1u << R) - 1u) << O;
    const uint32_t v = lop3<kAndOr>(w, x2(m), 0x43004300u);
    constexpr uint32_t mul = x2(bf16_bits(1, O));
    constexpr uint32_t add = x2(bf16_bits(-((128 >> O) + (1 << (R - 1))), 0));
    return hfma2(v, mul, add);
}

// Field of R bits at offset O, magic-encoded only: bf16 128 + field * 2^O.
// The GEMV folds the 2^-O into a pre-scaled activation copy and the
// (128 * 2^-O + z) zero point into a per-group constant (zp_off<R> below).
template <int R, int O>
MQ_HD uint32_t field_raw(uint32_t w) {
    static_assert(O + R <= 7, "field must sit inside the bf16 mantissa");
    constexpr uint32_t m = ((1u << R) - 1u) << O;
    return lop3<kAndOr>(w, x2(m), 0x43004300u);
}
template <int R, int O, bool RAW>
MQ_HD uint32_t field_out(uint32_t w) {
    if constexpr (RAW) return field_raw<R, O>(w);
    else return field_bf16<R, O>(w);
}

// 8-bit field at offset 0 (bit 7 would land in the bf16 exponent):
// (low7 | 0x4300) - (bit7 ? 128 : 256) = code - 128, exact.
MQ_HD uint32_t field8_bf16(uint32_t w) {
    const uint32_t a = lop3<kAndOr>(w, 0x007F007Fu, 0x43004300u);
    const uint32_t b = lop3<kAndXor>(w, 0x00800080u, 0x43804380u);
    return hsub2(a, b);
}

// ----------------------------------------------------------------------------
// Bitsliced rounding slice (slicing.py:31-48), 32 weights per instruction.
// T[0..R-1] = top R code bits (T[0] = MSB), T[R] = the rounding bit k-1.
//   carry = T[R] & ~(T[0] & ... & T[R-1])      (clamp: no carry into all-ones)
//   S = T + carry  (ripple from the LSB; cannot overflow because of the clamp)
// This is exactly min((q + 2^(k-1)) >> k, 2^r - 1) (finding 1;
// exhaustively checked in tests/test_oracle.py::test_slice_decomposition_identity
// and on device by tests/test_gpu_parity.py).
template <int R>
MQ_HD void slice_bitsliced(const uint32_t (&T)[R + 1], uint32_t (&S)[R]) {
    uint32_t all = T[0];
#pragma unroll
    for (int j = 1; j < R; ++j) all &= T[j];
    uint32_t c = T[R] & ~all;
#pragma unroll
    for (int j = R - 1; j >= 0; --j) {
        S[j] = T[j] ^ c;
        c &= T[j];
    }
}

// ----------------------------------------------------------------------------
// Plane -> field transpose networks.  Input P[0..NP-1] LSB-plane first.
// After the network, word W_i holds, in field f (f-th NP-bit field of the
// word), the NP-bit value of the weight at bit position NP*f + i.  Each stage
// is a masked exchange of bit blocks between two words (2 shifts + 2 LOP3).
template <int S>
MQ_HD void xchg(uint32_t& a, uint32_t& b, uint32_t m) {
    const uint32_t na = lop3<kSelect>(a, shl<S>(b), m);
    const uint32_t nb = lop3<kSelect>(shr<S>(a), b, m);
    a = na;
    b = nb;
}
template <int NP>
MQ_HD void transpose_planes(uint32_t (&P)[NP]) {
    if constexpr (NP == 8) {
#pragma unroll
        for (int j = 0; j < 4; ++j) xchg<4>(P[j], P[j + 4], 0x0F0F0F0Fu);
    }
    if constexpr (NP >= 4) {
#pragma unroll
        for (int j0 = 0; j0 < NP; j0 += 4) {
            xchg<2>(P[j0 + 0], P[j0 + 2], 0x33333333u);
            xchg<2>(P[j0 + 1], P[j0 + 3], 0x33333333u);
        }
    }
#pragma unroll
    for (int j = 0; j < NP; j += 2) xchg<1>(P[j], P[j + 1], 0x55555555u);
}

// ----------------------------------------------------------------------------
// Decode one lane word-set into the 16 bf16x2 A registers of four mma k16
// steps: A[p] holds weights at bit positions p (low half) and p + 16 (high
// half) as exact bf16 (s - 2^(R-1)).  S[0..R-1] are the sliced planes, MSB
// first.
template <int R, bool RAW = false>
MQ_HD void decode_word(const uint32_t (&S)[R], uint32_t (&A)[16]) {
    if constexpr (R == 2) {
        uint32_t P[2] = {S[1], S[0]};
        transpose_planes<2>(P);
        // W_i field n (offset 2n) <-> position 2n + i
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const uint32_t w0 = P[i], w6 = shr_x<6>(P[i]), w12 = shr_x<12>(P[i]);
            A[0 + i] = field_out<2, 0, RAW>(w0);
            A[2 + i] = field_out<2, 2, RAW>(w0);
            A[4 + i] = field_out<2, 4, RAW>(w0);
            A[6 + i] = field_out<2, 0, RAW>(w6);
            A[8 + i] = field_out<2, 2, RAW>(w6);
            A[10 + i] = field_out<2, 4, RAW>(w6);
            A[12 + i] = field_out<2, 0, RAW>(w12);
            A[14 + i] = field_out<2, 2, RAW>(w12);
        }
    } else if constexpr (R == 3 || R == 4) {
        uint32_t P[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) P[j] = j < R ? S[R - 1 - j] : 0u;
        transpose_planes<4>(P);
        // W_i nibble n (offset 4n) <-> position 4n + i
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t w = P[i];
            if constexpr (R == 3) {
                const uint32_t w8 = shr_x<8>(w);
                A[0 + i] = field_out<3, 0, RAW>(w);
                A[4 + i] = field_out<3, 4, RAW>(w);
                A[8 + i] = field_out<3, 0, RAW>(w8);
                A[12 + i] = field_out<3, 4, RAW>(w8);
            } else {
                A[0 + i] = field_out<4, 0, RAW>(w);
                A[4 + i] = field_out<4, 3, RAW>(shr_x<1>(w));
                A[8 + i] = field_out<4, 0, RAW>(shr_x<8>(w));
                A[12 + i] = field_out<4, 3, RAW>(shr_x<9>(w));
            }
        }
    } else {
        static_assert(R == 6 || R == 8, "R must be on the ladder {2,3,4,6,8}");
        uint32_t P[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) P[j] = j < R ? S[R - 1 - j] : 0u;
        transpose_planes<8>(P);
        // W_i byte b (offset 8b) <-> position 8b + i
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (R == 6) {
                A[0 + i] = field_out<6, 0, RAW>(P[i]);
                A[8 + i] = field_out<6, 0, RAW>(shr_x<8>(P[i]));
            } else {
                A[0 + i] = field8_bf16(P[i]);
                A[8 + i] = field8_bf16(shr_x<8>(P[i]));
            }
        }
    }
}

// ---- fp16 raw decode (r in {4, 8}) -------------------------------------------
// fp16 has a 10-bit mantissa, so (w & mask) | 0x6400 = fp16 1024 + field * 2^o is
// exact for o + r <= 10: a nibble fits at offsets 0 AND 4 of each half (one
// byte shift per word instead of three), a whole byte at offset 0 (one LOP3
// per register instead of two LOP3 + HSUB2).  Used with fp16 activations.
template <int R, int O>
MQ_HD uint32_t field_raw16(uint32_t w) {
    static_assert(O + R <= 10, "field must sit inside the fp16 mantissa");
    constexpr uint32_t m = ((1u << R) - 1u) << O;
    return lop3<kAndOr>(w, x2(m), 0x64006400u);
}
template <int R>
MQ_HD void decode_word_f16(const uint32_t (&S)[R], uint32_t (&A)[16]) {
    static_assert(R == 4 || R == 8, "fp16 decode serves r in {4, 8}");
    if constexpr (R == 4) {
        uint32_t P[4] = {S[3], S[2], S[1], S[0]};
        transpose_planes<4>(P);
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // nibble n of W_i <-> bit position 4n + i
            const uint32_t w = P[i], w8 = shr_x<8>(P[i]);
            A[0 + i] = field_raw16<4, 0>(w);
            A[4 + i] = field_raw16<4, 4>(w);
            A[8 + i] = field_raw16<4, 0>(w8);
            A[12 + i] = field_raw16<4, 4>(w8);
        }
    } else {
        uint32_t P[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) P[j] = S[7 - j];
        transpose_planes<8>(P);
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // byte b of W_i <-> bit position 8b + i
            A[0 + i] = field_raw16<8, 0>(P[i]);
            A[8 + i] = field_raw16<8, 0>(shr_x<8>(P[i]));
        }
    }
}
// fp16 field offset of k16 step s (same for both 8-column halves)
template <int R>
__host__ __device__ constexpr int zp_off16(int s) { return (R == 4 && (s & 1)) ? 4 : 0; }

// Zero-point folding for the raw decode (R in {2,3,4,6}).  decode_word<R, true>
// leaves A[4s+q] = bf16(128 + s_code * 2^o) with o = kOff[s][q >> 1] (the field
// offset of k16 step s, 8-column half q >> 1).  The GEMV multiplies that half
// by an activation copy scaled by 2^-o, so the MMA returns
//   sum (s_code - z) x + sum (128 * 2^-o + z) x,
// and subtracts the second term, computed per scale group by the same MMA
// chain on the all-zero-code A fragment kZeroA (so zero-code rows are exactly
// 0, as in the reference, test_matmul.py:61-66).
template <int R>
__host__ __device__ constexpr int zp_off(int s, int h) {
    // R = 2: W_i fields n = 2s + h at offsets 0,2,4 | 0 (>>6),2,4 | 0 (>>12),2
    // R = 3: nibble n = s at offsets 0,4 | 0 (>>8),4      R = 4: 0, 3 (>>1) | 0 (>>8), 3 (>>9)
    // R = 6, 8: byte fields at offset 0
    return R == 2 ? ((2 * s + h) % 3 == 0 ? 0 : ((2 * s + h) % 3 == 1 ? 2 : 4))
         : R == 3 ? ((s & 1) ? 4 : 0)
         : R == 4 ? ((s & 1) ? 3 : 0)
         : 0;
}
// distinct offsets -> activation copy index (copy c is x * 2^-zp_copy_off(R, c))
__host__ __device__ constexpr int zp_copy_of(int R, int o) {
    return o == 0 ? 0 : (R == 2 ? (o == 2 ? 1 : 2) : 1);
}
__host__ __device__ constexpr int zp_ncopies(int R) { return R == 2 ? 3 : (R == 3 || R == 4 ? 2 : 1); }
__host__ __device__ constexpr int zp_copy_off(int R, int c) {
    return c == 0 ? 0 : (R == 2 ? (c == 1 ? 2 : 4) : (R == 3 ? 4 : 3));
}
// A register (s, q) of the all-zero-code fragment: 128 + z * 2^o, both halves
template <int R>
__host__ __device__ constexpr uint32_t zp_zero_a(int s, int q) {
    return x2(bf16_bits(128 + ((1 << (R - 1)) << zp_off<R>(s, q >> 1)), 0));
}

// Loaded planes -> sliced planes.  CHILD: planes already hold the r-bit code
// (mode C, r planes).  Parent mode P: R+1 planes (top R + rounding bit), or
// 8 planes at R = 8 (identity slice).
template <int R, bool CHILD>
struct PlaneCount {
    static constexpr int value = CHILD ? R : (R < 8 ? R + 1 : 8);
};

template <int R, bool CHILD>
MQ_HD void slice_loaded(const uint32_t (&T)[PlaneCount<R, CHILD>::value],
                                             uint32_t (&S)[R]) {
    if constexpr (CHILD || R == 8) {
#pragma unroll
        for (int j = 0; j < R; ++j) S[j] = T[j];
    } else {
        slice_bitsliced<R>(T, S);
    }
}

// ----------------------------------------------------------------------------
// Memory / tensor-core wrappers.
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t word_of(const uint4& v, int w) {
    return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&d)[4], uint32_t saddr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
                 : "r"(saddr));
}

// D += A * B, m16n8k16, bf16 inputs, fp32 accumulate.
__device__ __forceinline__ void mma_acc(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                        uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// fp16 variant: D += A * B, m16n8k16, f16 inputs, fp32 accumulate.
__device__ __forceinline__ void mma_acc_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                            uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_zero_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                             uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%10,%10,%10,%10};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.0f));
}
// D = A * B (zero accumulator input).
__device__ __forceinline__ void mma_zero(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%10,%10,%10,%10};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.0f));
}

__device__ __forceinline__ float bf16_to_f32(uint16_t h) {
    return __uint_as_float(((uint32_t)h) << 16);
}
__device__ __forceinline__ uint16_t f32_to_bf16_rn(float f) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// ---- TMA bulk copies + mbarriers (per-warp staging ring) --------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
// ---- CTA-pair split-K (cluster of 2): chunk 1's CTA ships its finished
// tile partial into chunk 0's shared memory with st.async, which completes
// bytes on chunk 0's per-tile mbarrier -- no global partials, no tickets.
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float a, float b, float c, float d, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                 ::"r"(raddr), "f"(a), "f"(b), "f"(c), "f"(d), "r"(rbar) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ float lds32f(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ int ld_acquire_s32(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// Programmatic dependent launch controls (no-ops when launched without PDL).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;");
}

}  // namespace mq
