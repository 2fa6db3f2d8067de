// matq_aux.cu -- K1 (parent/child plane pack), K2 (slice / decode / dequant /
// child materialisation) and the format/compat kernels behind the drop-in
// API (elementwise slice_code, float64 dequant, exact matmul_ref, the
// reference's own child bit-plane layout).  None of these is on the decode
// hot path except through the shared device functions in matq_common.cuh,
// which K2 exercises exactly as K3 uses them.
#include "matq_common.cuh"
#include "matq_internal.h"

#include <algorithm>

namespace mq {

// ---------------------------------------------------------------------------
// K1: codes (N, K) uint8 with `nbits` significant bits -> MSB-first planes in
// the step-interleaved blob.  One thread per (row tile, step, lane, word).
__global__ void k_pack_planes(const uint8_t* __restrict__ codes, long long ldc, Layout L, int nbits,
                              uint32_t* __restrict__ blob) {
    const long long total = (long long)L.n_rt * L.nsteps * 128;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(idx & 3), lane = (int)((idx >> 2) & 31);
        const long long blk = idx >> 7;
        const int st = (int)(blk % L.nsteps), rt = (int)(blk / L.nsteps);
        uint32_t words[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
        for (int bit = 0; bit < 32; ++bit) {
            int ro, co;
            word_bit_pos(lane, w, bit, ro, co);
            const int row = rt * kTileRows + ro, col = st * kStepCols + co;
            const uint32_t q = (row < L.N && col < L.K) ? codes[(long long)row * ldc + col] : 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < nbits) words[j] |= ((q >> (nbits - 1 - j)) & 1u) << bit;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < nbits) blob[L.plane_word(rt, st, j, lane, w)] = words[j];
    }
}

// Group scales (N, ng) row-major (QuantGrid.scales, grid.py:75) -> the
// blob's per-step scale blocks (spg > 0) and/or the tiled array
// [Np/16][ngp][16] (generic group sizes).  Padding entries are 0.
__global__ void k_pack_scales(const float* __restrict__ scales, Layout L, int ng,
                              uint32_t* __restrict__ blob, float* __restrict__ ts) {
    if (blob && L.spg > 0) {
        const long long total = (long long)L.n_rt * L.nsteps * L.spg * 16;
        for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
             idx += (long long)gridDim.x * blockDim.x) {
            const int r16 = (int)(idx & 15);
            const long long rest = idx >> 4;
            const int gi = (int)(rest % L.spg);
            const long long blk = rest / L.spg;
            const int st = (int)(blk % L.nsteps), rt = (int)(blk / L.nsteps);
            const int row = rt * 16 + r16;
            const int grp = (st * kStepCols + gi * min(L.G, kStepCols)) / L.G;
            const float v = (row < L.N && grp < ng) ? scales[(long long)row * ng + grp] : 0.0f;
            blob[L.block(rt, st) + gi * 16 + r16] = __float_as_uint(v);
        }
    }
    if (ts) {
        const long long total = (long long)L.Np * L.ngp;
        for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
             idx += (long long)gridDim.x * blockDim.x) {
            const int r16 = (int)(idx & 15);
            const long long rest = idx >> 4;
            const int grp = (int)(rest % L.ngp), rt = (int)(rest / L.ngp);
            const int row = rt * 16 + r16;
            ts[idx] = (row < L.N && grp < ng) ? scales[(long long)row * ng + grp] : 0.0f;
        }
    }
}

__device__ __forceinline__ float layout_scale(const Layout& L, const uint32_t* blob, const float* ts,
                                              int rt, int st, int r16, int col_in_step) {
    if (L.spg > 0) return __uint_as_float(blob[L.scale_word(rt, st, r16, col_in_step)]);
    const int grp = (st * kStepCols + col_in_step) / L.G;
    return ts[((long long)rt * L.ngp + grp) * 16 + r16];
}

// ---------------------------------------------------------------------------
// K2a: blob -> r-bit sliced codes (N, K) via the bitsliced slice K3 uses.
template <int R, bool CHILD>
__global__ void k_slice_codes(const uint32_t* __restrict__ blob, Layout L, uint8_t* __restrict__ out,
                              long long ldo) {
    constexpr int NPL = PlaneCount<R, CHILD>::value;
    const long long total = (long long)L.n_rt * L.nsteps * 128;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(idx & 3), lane = (int)((idx >> 2) & 31);
        const long long blk = idx >> 7;
        const int st = (int)(blk % L.nsteps), rt = (int)(blk / L.nsteps);
        uint32_t T[NPL];
#pragma unroll
        for (int j = 0; j < NPL; ++j) T[j] = blob[L.plane_word(rt, st, j, lane, w)];
        uint32_t S[R];
        slice_loaded<R, CHILD>(T, S);
        for (int bit = 0; bit < 32; ++bit) {
            int ro, co;
            word_bit_pos(lane, w, bit, ro, co);
            const int row = rt * kTileRows + ro, col = st * kStepCols + co;
            if (row >= L.N || col >= L.K) continue;
            uint32_t q = 0;
#pragma unroll
            for (int j = 0; j < R; ++j) q |= ((S[j] >> bit) & 1u) << (R - 1 - j);
            out[(long long)row * ldo + col] = (uint8_t)q;
        }
    }
}

// K2b: blob -> dequantised weights through the exact K3 decode path
// (bitsliced slice + transpose network + bf16 magic conversion).
//   vals (int8, optional): s - 2^(r-1) as decoded in bf16 registers
//   W (fp32, optional): (s - z) * (scale * out_scale), one fp32 rounding --
//   the same arithmetic as PackedLayer.dense_f32 (matmul.py:64-69).
template <int R, bool CHILD>
__global__ void k_decode_dense(const uint32_t* __restrict__ blob, const float* __restrict__ ts,
                               Layout L, float out_scale, int8_t* __restrict__ vals,
                               float* __restrict__ W, long long ldw) {
    constexpr int NPL = PlaneCount<R, CHILD>::value;
    const long long total = (long long)L.n_rt * L.nsteps * 128;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(idx & 3), lane = (int)((idx >> 2) & 31);
        const long long blk = idx >> 7;
        const int st = (int)(blk % L.nsteps), rt = (int)(blk / L.nsteps);
        uint32_t T[NPL];
#pragma unroll
        for (int j = 0; j < NPL; ++j) T[j] = blob[L.plane_word(rt, st, j, lane, w)];
        uint32_t S[R];
        slice_loaded<R, CHILD>(T, S);
        uint32_t A[16];
        decode_word<R>(S, A);
#pragma unroll
        for (int p = 0; p < 16; ++p) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                int ro, co;
                word_bit_pos(lane, w, p + 16 * h, ro, co);
                const int row = rt * kTileRows + ro, col = st * kStepCols + co;
                if (row >= L.N || col >= L.K) continue;
                const float v = bf16_to_f32((uint16_t)(A[p] >> (16 * h)));
                if (vals) vals[(long long)row * ldw + col] = (int8_t)v;
                if (W) W[(long long)row * ldw + col] = v * (layout_scale(L, blob, ts, rt, st, ro, co) * out_scale);
            }
        }
    }
}

// K2c: mode C child materialisation: parent blob -> r-plane child blob
// (scale blocks copied, planes sliced).
template <int R>
__global__ void k_materialize_child(const uint32_t* __restrict__ blob, Layout Lp, Layout Lc,
                                    uint32_t* __restrict__ child) {
    const long long nwords = (long long)Lp.n_rt * Lp.nsteps * 128;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < nwords;
         idx += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(idx & 3), lane = (int)((idx >> 2) & 31);
        const long long blk = idx >> 7;
        const int st = (int)(blk % Lp.nsteps), rt = (int)(blk / Lp.nsteps);
        constexpr int NPL = PlaneCount<R, false>::value;
        uint32_t T[NPL];
#pragma unroll
        for (int j = 0; j < NPL; ++j) T[j] = blob[Lp.plane_word(rt, st, j, lane, w)];
        uint32_t S[R];
        slice_loaded<R, false>(T, S);
#pragma unroll
        for (int j = 0; j < R; ++j) child[Lc.plane_word(rt, st, j, lane, w)] = S[j];
        if (lane * 4 + w < 16 * Lp.spg)  // copy the step's scale block
            child[Lc.block(rt, st) + lane * 4 + w] = blob[Lp.block(rt, st) + lane * 4 + w];
    }
}

// ---------------------------------------------------------------------------
// Elementwise slice_code / slice_to_code (slicing.py:31-54) for any 2<=c<=8.
__global__ void k_slice_elementwise(const uint8_t* __restrict__ q, long long n, int c, int r,
                                    int on_master, uint8_t* __restrict__ out, int* err) {
    const int k = c - r, qmax = (1 << c) - 1;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        int v = q[i];
        if (v > qmax) {
            atomicOr(err, 1);
            continue;
        }
        if (k > 0) {
            v = min((v + (1 << (k - 1))) >> k, (1 << r) - 1);
            if (on_master) v <<= k;
        }
        out[i] = (uint8_t)v;
    }
}

// grid.py:128-149 (dequant_value / dequant) in float64:
// scale[row, col // G] * (2^(c-r) * (code - 2^(r-1))).
__global__ void k_dequant_f64(const uint8_t* __restrict__ codes, int N, int K,
                              const float* __restrict__ scales, int ng, int G, int c, int r,
                              double* __restrict__ out, int* err) {
    const long long total = (long long)N * K;
    const long long step = 1ll << (c - r), zr = 1ll << (r - 1);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(i / K), col = (int)(i - (long long)row * K);
        const int q = codes[i];
        if (q > (1 << r) - 1) {
            atomicOr(err, 1);
            continue;
        }
        const double s = (double)scales[(long long)row * ng + col / G];
        out[i] = s * (double)(step * ((long long)q - zr));
    }
}

// grid.py:128-140 dequant_value with a per-element float64 scale.
__global__ void k_dequant_value_f64(const uint8_t* __restrict__ q, const double* __restrict__ scale,
                                    long long n, int c, int r, double* __restrict__ out, int* err) {
    const long long step = 1ll << (c - r), zr = 1ll << (r - 1);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int v = q[i];
        if (v > (1 << r) - 1) {
            atomicOr(err, 1);
            continue;
        }
        out[i] = scale[i] * (double)(step * ((long long)v - zr));
    }
}

// matmul.py:85-92 matmul_ref, bit-exact on device: float32 product then
// float32 add, k ascending (explicit _rn intrinsics forbid FMA contraction).
__global__ void k_matmul_ref(const float* __restrict__ X, int B, int K,
                             const float* __restrict__ W, int N, float* __restrict__ Y) {
    const long long total = (long long)B * N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(i / N), n = (int)(i - (long long)b * N);
        const float* x = X + (long long)b * K;
        const float* w = W + (long long)n * K;
        float y = 0.0f;
        for (int k = 0; k < K; ++k) y = __fadd_rn(y, __fmul_rn(x[k], w[k]));
        Y[i] = y;
    }
}

// The reference's child bit-plane layout (packing.py:81-126): base uint64
// (bits 0..1 of weight i at [2i, 2i+1]), uint32 planes for bits 2 and 3.
__global__ void k_pack_ref_layout(const uint8_t* __restrict__ codes, int N, int K, int bits,
                                  unsigned long long* __restrict__ base, uint32_t* __restrict__ b2,
                                  uint32_t* __restrict__ b3, int* err) {
    const int nu = (K + 31) / 32;
    const long long total = (long long)N * nu;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(i / nu), u = (int)(i - (long long)row * nu);
        unsigned long long wb = 0;
        uint32_t p2 = 0, p3 = 0;
        for (int l = 0; l < 32; ++l) {
            const int col = u * 32 + l;
            const uint32_t q = col < K ? codes[(long long)row * K + col] : 0u;
            if (q >= (1u << bits)) atomicOr(err, 1);
            wb |= (unsigned long long)(q & 3u) << (2 * l);
            p2 |= ((q >> 2) & 1u) << l;
            p3 |= ((q >> 3) & 1u) << l;
        }
        base[i] = wb;
        if (b2) b2[i] = p2;
        if (b3) b3[i] = p3;
    }
}

__global__ void k_unpack_ref_layout(const unsigned long long* __restrict__ base,
                                    const uint32_t* __restrict__ b2, const uint32_t* __restrict__ b3,
                                    int N, int K, uint8_t* __restrict__ codes) {
    const int nu = (K + 31) / 32;
    const long long total = (long long)N * K;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(i / K), col = (int)(i - (long long)row * K);
        const long long wi = (long long)row * nu + col / 32;
        const int l = col & 31;
        uint32_t q = (uint32_t)((base[wi] >> (2 * l)) & 3ull);
        if (b2) q |= ((b2[wi] >> l) & 1u) << 2;
        if (b3) q |= ((b3[wi] >> l) & 1u) << 3;
        codes[i] = (uint8_t)q;
    }
}

// ---------------------------------------------------------------------------
// launch helpers used by matq_abi.cu
static inline int grid_for(long long n, int block = 256) {
    long long g = (n + block - 1) / block;
    if (g > 148LL * 32) g = 148LL * 32;
    if (g < 1) g = 1;
    return (int)g;
}

cudaError_t launch_pack_planes(const uint8_t* codes, long long ldc, const Layout& L, int nbits,
                               uint32_t* blob, cudaStream_t s) {
    const long long total = (long long)L.n_rt * L.nsteps * 128;
    k_pack_planes<<<grid_for(total), 256, 0, s>>>(codes, ldc, L, nbits, blob);
    return cudaGetLastError();
}

cudaError_t launch_pack_scales(const float* scales, const Layout& L, int ng, uint32_t* blob, float* ts,
                               cudaStream_t s) {
    const long long total = std::max((long long)L.n_rt * L.nsteps * L.spg * 16, (long long)L.Np * L.ngp);
    k_pack_scales<<<grid_for(total), 256, 0, s>>>(scales, L, ng, blob, ts);
    return cudaGetLastError();
}

template <bool CHILD>
static cudaError_t slice_codes_dispatch(int r, const uint32_t* blob, const Layout& L, uint8_t* out,
                                        long long ldo, cudaStream_t s) {
    const int gr = grid_for((long long)L.n_rt * L.nsteps * 128);
    switch (r) {
        case 2: k_slice_codes<2, CHILD><<<gr, 256, 0, s>>>(blob, L, out, ldo); break;
        case 3: k_slice_codes<3, CHILD><<<gr, 256, 0, s>>>(blob, L, out, ldo); break;
        case 4: k_slice_codes<4, CHILD><<<gr, 256, 0, s>>>(blob, L, out, ldo); break;
        case 6: k_slice_codes<6, CHILD><<<gr, 256, 0, s>>>(blob, L, out, ldo); break;
        case 8: k_slice_codes<8, CHILD><<<gr, 256, 0, s>>>(blob, L, out, ldo); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_slice_codes(int r, bool child, const uint32_t* blob, const Layout& L, uint8_t* out,
                               long long ldo, cudaStream_t s) {
    return child ? slice_codes_dispatch<true>(r, blob, L, out, ldo, s)
                 : slice_codes_dispatch<false>(r, blob, L, out, ldo, s);
}

template <bool CHILD>
static cudaError_t decode_dispatch(int r, const uint32_t* blob, const float* ts, const Layout& L,
                                   float os, int8_t* vals, float* W, long long ldw, cudaStream_t s) {
    const int gr = grid_for((long long)L.n_rt * L.nsteps * 128);
#define MQ_DD(R_) k_decode_dense<R_, CHILD><<<gr, 256, 0, s>>>(blob, ts, L, os, vals, W, ldw)
    switch (r) {
        case 2: MQ_DD(2); break;
        case 3: MQ_DD(3); break;
        case 4: MQ_DD(4); break;
        case 6: MQ_DD(6); break;
        case 8: MQ_DD(8); break;
        default: return cudaErrorInvalidValue;
    }
#undef MQ_DD
    return cudaGetLastError();
}

cudaError_t launch_decode_dense(int r, bool child, const uint32_t* blob, const float* ts,
                                const Layout& L, float out_scale, int8_t* vals, float* W,
                                long long ldw, cudaStream_t s) {
    return child ? decode_dispatch<true>(r, blob, ts, L, out_scale, vals, W, ldw, s)
                 : decode_dispatch<false>(r, blob, ts, L, out_scale, vals, W, ldw, s);
}

cudaError_t launch_materialize_child(int r, const uint32_t* blob, const Layout& Lp, uint32_t* child,
                                     cudaStream_t s) {
    const Layout Lc = Layout::make(Lp.N, Lp.K, Lp.G, r);
    const int gr = grid_for((long long)Lp.n_rt * Lp.nsteps * 128);
    switch (r) {
        case 2: k_materialize_child<2><<<gr, 256, 0, s>>>(blob, Lp, Lc, child); break;
        case 3: k_materialize_child<3><<<gr, 256, 0, s>>>(blob, Lp, Lc, child); break;
        case 4: k_materialize_child<4><<<gr, 256, 0, s>>>(blob, Lp, Lc, child); break;
        case 6: k_materialize_child<6><<<gr, 256, 0, s>>>(blob, Lp, Lc, child); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_slice_elementwise(const uint8_t* q, long long n, int c, int r, int on_master,
                                     uint8_t* out, int* err, cudaStream_t s) {
    k_slice_elementwise<<<grid_for(n), 256, 0, s>>>(q, n, c, r, on_master, out, err);
    return cudaGetLastError();
}

cudaError_t launch_dequant_f64(const uint8_t* codes, int N, int K, const float* scales, int ng,
                               int G, int c, int r, double* out, int* err, cudaStream_t s) {
    k_dequant_f64<<<grid_for((long long)N * K), 256, 0, s>>>(codes, N, K, scales, ng, G, c, r, out,
                                                             err);
    return cudaGetLastError();
}

cudaError_t launch_dequant_value_f64(const uint8_t* q, const double* scale, long long n, int c,
                                     int r, double* out, int* err, cudaStream_t s) {
    k_dequant_value_f64<<<grid_for(n), 256, 0, s>>>(q, scale, n, c, r, out, err);
    return cudaGetLastError();
}

cudaError_t launch_matmul_ref(const float* X, int B, int K, const float* W, int N, float* Y,
                              cudaStream_t s) {
    k_matmul_ref<<<grid_for((long long)B * N, 128), 128, 0, s>>>(X, B, K, W, N, Y);
    return cudaGetLastError();
}

cudaError_t launch_pack_ref_layout(const uint8_t* codes, int N, int K, int bits,
                                   unsigned long long* base, uint32_t* b2, uint32_t* b3, int* err,
                                   cudaStream_t s) {
    const long long total = (long long)N * ((K + 31) / 32);
    k_pack_ref_layout<<<grid_for(total), 256, 0, s>>>(codes, N, K, bits, base, b2, b3, err);
    return cudaGetLastError();
}

cudaError_t launch_unpack_ref_layout(const unsigned long long* base, const uint32_t* b2,
                                     const uint32_t* b3, int N, int K, uint8_t* codes,
                                     cudaStream_t s) {
    k_unpack_ref_layout<<<grid_for((long long)N * K), 256, 0, s>>>(base, b2, b3, N, K, codes);
    return cudaGetLastError();
}

}  // namespace mq
