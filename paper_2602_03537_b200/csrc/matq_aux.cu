// matq_aux.cu -- K1 (parent/child plane pack), K2 (slice / decode / dequant /
// child materialisation) and the format/compat kernels behind the drop-in
// API (elementwise slice_code, float64 dequant, exact matmul_ref, the
// reference's own child bit-plane layout).  None of these is on the decode
// hot path except through the shared device functions in matq_common.cuh,
// which K2 exercises exactly as K3 uses them.
#include "matq_common.cuh"
#include "matq_internal.h"

namespace mq {

// ---------------------------------------------------------------------------
// K1: codes (N, K) uint8 with `nbits` significant bits -> MSB-first planes.
// One thread per (row tile, step, lane, word); each writes nbits words.
__global__ void k_pack_planes(const uint8_t* __restrict__ codes, long long ldc, int N, int K,
                              int nbits, uint32_t* __restrict__ planes, long long plane_stride,
                              int n_rt, int nsteps) {
    const long long total = (long long)n_rt * nsteps * 128;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(idx & 3), lane = (int)((idx >> 2) & 31);
        const long long blk = idx >> 7;
        const int st = (int)(blk % nsteps), rt = (int)(blk / nsteps);
        uint32_t words[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
        for (int bit = 0; bit < 32; ++bit) {
            int ro, co;
            word_bit_pos(lane, w, bit, ro, co);
            const int row = rt * kTileRows + ro, col = st * kStepCols + co;
            const uint32_t q = (row < N && col < K) ? codes[(long long)row * ldc + col] : 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < nbits) words[j] |= ((q >> (nbits - 1 - j)) & 1u) << bit;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < nbits) planes[j * plane_stride + idx] = words[j];
    }
}

// scales (N, ng) row-major (QuantGrid.scales, grid.py:293) -> tiled
// [Np/16][ngp][16]; padding entries are 0 (their activations are 0 too).
__global__ void k_tile_scales(const float* __restrict__ scales, int N, int ng, int ngp, int Np,
                              float* __restrict__ ts) {
    const long long total = (long long)Np * ngp;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int r16 = (int)(idx & 15);
        const long long rest = idx >> 4;
        const int grp = (int)(rest % ngp), rt = (int)(rest / ngp);
        const int row = rt * 16 + r16;
        ts[idx] = (row < N && grp < ng) ? scales[(long long)row * ng + grp] : 0.0f;
    }
}

// ---------------------------------------------------------------------------
// K2a: planes -> r-bit sliced codes (N, K) via the bitsliced slice K3 uses.
template <int R, bool CHILD>
__global__ void k_slice_codes(const uint32_t* __restrict__ planes, long long plane_stride, int N,
                              int K, int n_rt, int nsteps, uint8_t* __restrict__ out, long long ldo) {
    constexpr int NPL = PlaneCount<R, CHILD>::value;
    const long long total = (long long)n_rt * nsteps * 128;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(idx & 3), lane = (int)((idx >> 2) & 31);
        const long long blk = idx >> 7;
        const int st = (int)(blk % nsteps), rt = (int)(blk / nsteps);
        uint32_t T[NPL];
#pragma unroll
        for (int j = 0; j < NPL; ++j) T[j] = planes[j * plane_stride + idx];
        uint32_t S[R];
        slice_loaded<R, CHILD>(T, S);
        for (int bit = 0; bit < 32; ++bit) {
            int ro, co;
            word_bit_pos(lane, w, bit, ro, co);
            const int row = rt * kTileRows + ro, col = st * kStepCols + co;
            if (row >= N || col >= K) continue;
            uint32_t q = 0;
#pragma unroll
            for (int j = 0; j < R; ++j) q |= ((S[j] >> bit) & 1u) << (R - 1 - j);
            out[(long long)row * ldo + col] = (uint8_t)q;
        }
    }
}

// K2b: planes -> dequantised weights through the exact K3 decode path
// (bitsliced slice + transpose network + bf16 magic conversion).
//   vals (int8, optional): s - 2^(r-1) as decoded in bf16 registers
//   W (fp32, optional): (s - z) * (scale * out_scale), one fp32 rounding --
//   the same arithmetic as PackedLayer.dense_f32 (matmul.py:232-237).
template <int R, bool CHILD>
__global__ void k_decode_dense(const uint32_t* __restrict__ planes, long long plane_stride,
                               const float* __restrict__ tscales, int ngp, int G, float out_scale,
                               int N, int K, int n_rt, int nsteps, int8_t* __restrict__ vals,
                               float* __restrict__ W, long long ldw) {
    constexpr int NPL = PlaneCount<R, CHILD>::value;
    const long long total = (long long)n_rt * nsteps * 128;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(idx & 3), lane = (int)((idx >> 2) & 31);
        const long long blk = idx >> 7;
        const int st = (int)(blk % nsteps), rt = (int)(blk / nsteps);
        uint32_t T[NPL];
#pragma unroll
        for (int j = 0; j < NPL; ++j) T[j] = planes[j * plane_stride + idx];
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
                if (row >= N || col >= K) continue;
                const float v = bf16_to_f32((uint16_t)(A[p] >> (16 * h)));
                if (vals) vals[(long long)row * ldw + col] = (int8_t)v;
                if (W) {
                    const float sc = tscales[((long long)rt * ngp + col / G) * 16 + ro] * out_scale;
                    W[(long long)row * ldw + col] = v * sc;
                }
            }
        }
    }
}

// K2c: mode C child materialisation: parent planes -> r sliced planes.
template <int R>
__global__ void k_materialize_child(const uint32_t* __restrict__ planes, long long plane_stride,
                                    long long nwords, uint32_t* __restrict__ child,
                                    long long child_stride) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < nwords;
         idx += (long long)gridDim.x * blockDim.x) {
        constexpr int NPL = PlaneCount<R, false>::value;
        uint32_t T[NPL];
#pragma unroll
        for (int j = 0; j < NPL; ++j) T[j] = planes[j * plane_stride + idx];
        uint32_t S[R];
        slice_loaded<R, false>(T, S);
#pragma unroll
        for (int j = 0; j < R; ++j) child[j * child_stride + idx] = S[j];
    }
}

// ---------------------------------------------------------------------------
// Elementwise slice_code / slice_to_code (slicing.py:67-90) for any 2<=c<=8.
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

// grid.py:346-367 (dequant_value / dequant) in float64:
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

// grid.py:346-358 dequant_value with a per-element float64 scale.
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

// matmul.py:253-260 matmul_ref, bit-exact on device: float32 product then
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

cudaError_t launch_pack_planes(const uint8_t* codes, long long ldc, int N, int K, int nbits,
                               uint32_t* planes, cudaStream_t s) {
    const int n_rt = pad16(N) / 16, nsteps = pad256(K) / 256;
    const long long total = (long long)n_rt * nsteps * 128;
    k_pack_planes<<<grid_for(total), 256, 0, s>>>(codes, ldc, N, K, nbits, planes, total, n_rt,
                                                  nsteps);
    return cudaGetLastError();
}

cudaError_t launch_tile_scales(const float* scales, int N, int ng, int ngp, float* ts,
                               cudaStream_t s) {
    const int Np = pad16(N);
    k_tile_scales<<<grid_for((long long)Np * ngp), 256, 0, s>>>(scales, N, ng, ngp, Np, ts);
    return cudaGetLastError();
}

template <bool CHILD>
static cudaError_t slice_codes_dispatch(int r, const uint32_t* planes, long long ps, int N, int K,
                                        int n_rt, int nsteps, uint8_t* out, long long ldo,
                                        cudaStream_t s) {
    const long long total = (long long)n_rt * nsteps * 128;
    const int gr = grid_for(total);
    switch (r) {
        case 2: k_slice_codes<2, CHILD><<<gr, 256, 0, s>>>(planes, ps, N, K, n_rt, nsteps, out, ldo); break;
        case 3: k_slice_codes<3, CHILD><<<gr, 256, 0, s>>>(planes, ps, N, K, n_rt, nsteps, out, ldo); break;
        case 4: k_slice_codes<4, CHILD><<<gr, 256, 0, s>>>(planes, ps, N, K, n_rt, nsteps, out, ldo); break;
        case 6: k_slice_codes<6, CHILD><<<gr, 256, 0, s>>>(planes, ps, N, K, n_rt, nsteps, out, ldo); break;
        case 8: k_slice_codes<8, CHILD><<<gr, 256, 0, s>>>(planes, ps, N, K, n_rt, nsteps, out, ldo); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_slice_codes(int r, bool child, const uint32_t* planes, int N, int K,
                               uint8_t* out, long long ldo, cudaStream_t s) {
    const int n_rt = pad16(N) / 16, nsteps = pad256(K) / 256;
    const long long ps = (long long)n_rt * nsteps * 128;
    return child ? slice_codes_dispatch<true>(r, planes, ps, N, K, n_rt, nsteps, out, ldo, s)
                 : slice_codes_dispatch<false>(r, planes, ps, N, K, n_rt, nsteps, out, ldo, s);
}

template <bool CHILD>
static cudaError_t decode_dispatch(int r, const uint32_t* planes, long long ps, const float* ts,
                                   int ngp, int G, float os, int N, int K, int n_rt, int nsteps,
                                   int8_t* vals, float* W, long long ldw, cudaStream_t s) {
    const long long total = (long long)n_rt * nsteps * 128;
    const int gr = grid_for(total);
#define MQ_DD(R_) k_decode_dense<R_, CHILD><<<gr, 256, 0, s>>>(planes, ps, ts, ngp, G, os, N, K, n_rt, nsteps, vals, W, ldw)
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

cudaError_t launch_decode_dense(int r, bool child, const uint32_t* planes, const float* ts, int G,
                                float out_scale, int N, int K, int8_t* vals, float* W,
                                long long ldw, cudaStream_t s) {
    const int n_rt = pad16(N) / 16, nsteps = pad256(K) / 256;
    const long long ps = (long long)n_rt * nsteps * 128;
    const int ngp = cdiv(pad256(K), G);
    return child ? decode_dispatch<true>(r, planes, ps, ts, ngp, G, out_scale, N, K, n_rt, nsteps,
                                         vals, W, ldw, s)
                 : decode_dispatch<false>(r, planes, ps, ts, ngp, G, out_scale, N, K, n_rt, nsteps,
                                          vals, W, ldw, s);
}

cudaError_t launch_materialize_child(int r, const uint32_t* planes, int N, int K, uint32_t* child,
                                     cudaStream_t s) {
    const int n_rt = pad16(N) / 16, nsteps = pad256(K) / 256;
    const long long nw = (long long)n_rt * nsteps * 128;
    const int gr = grid_for(nw);
    switch (r) {
        case 2: k_materialize_child<2><<<gr, 256, 0, s>>>(planes, nw, nw, child, nw); break;
        case 3: k_materialize_child<3><<<gr, 256, 0, s>>>(planes, nw, nw, child, nw); break;
        case 4: k_materialize_child<4><<<gr, 256, 0, s>>>(planes, nw, nw, child, nw); break;
        case 6: k_materialize_child<6><<<gr, 256, 0, s>>>(planes, nw, nw, child, nw); break;
        case 8: k_materialize_child<8><<<gr, 256, 0, s>>>(planes, nw, nw, child, nw); break;
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
