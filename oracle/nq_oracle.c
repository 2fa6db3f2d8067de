/* nq_oracle.c -- CPU restatement of the reference (nestquant) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under paper_2602_03537_b200/ links,
 * imports or calls this file; it is the checker used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs.  Every function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/nestquant/).
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against
 * golden vectors produced by importing the reference itself
 * (tests/golden/make_golden.py) and against the reference's own known-answer
 * tests (tests/test_slicing.py:18-31, test_packing.py:37-69,
 * test_grid.py:83-93 in the reference tree).
 *
 * Build with -ffp-contract=off: matmul_ref's numpy loop rounds the product
 * and the sum separately (matmul.py:90-91), an FMA would not.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#define OQ_OK 0
#define OQ_BAD_ARGS 1
#define OQ_CODE_RANGE 2

/* slicing.py:22-28 (_check_slice_args): 2 <= c <= 8, r <= c, r >= 2. */
int oq_check_slice_args(int c, int r) {
    if (c < 2 || c > 8) return OQ_BAD_ARGS;
    if (r > c) return OQ_BAD_ARGS;
    if (r < 2) return OQ_BAD_ARGS;
    return OQ_OK;
}

/* slicing.py:31-48 (slice_code): min((q + 2^(k-1)) >> k, 2^r - 1) << k with
 * k = c - r; identity when k == 0.  slicing.py:51-54 (slice_to_code) drops
 * the final << k.  `on_master` selects slice_code (1) or slice_to_code (0). */
int oq_slice(const uint8_t* q, int64_t n, int c, int r, int on_master, uint8_t* out) {
    int st = oq_check_slice_args(c, r);
    if (st) return st;
    const int k = c - r;
    const int qmax = (1 << c) - 1;
    for (int64_t i = 0; i < n; i++)
        if (q[i] > qmax) return OQ_CODE_RANGE; /* slicing.py:39-40 */
    for (int64_t i = 0; i < n; i++) {
        int v = q[i];
        if (k > 0) {
            v = (v + (1 << (k - 1))) >> k;
            if (v > (1 << r) - 1) v = (1 << r) - 1;
            if (on_master) v <<= k;
        }
        out[i] = (uint8_t)v;
    }
    return OQ_OK;
}

/* slicing.py:127 (slice_layer scales): scales * float32(2^(c-r)), exact. */
void oq_scale_eff(const float* scales, int64_t n, int c, int r, float* out) {
    const float f = (float)(1 << (c - r));
    for (int64_t i = 0; i < n; i++) out[i] = scales[i] * f;
}

/* grid.py:128-140 (dequant_value) + grid.py:143-149 (dequant): float64
 * scale * (2^(c-r) * (code - 2^(r-1))), scale expanded per column by
 * grid.py:95-98 (column_scales, col // G).  codes (N,K) r-bit, scales
 * (N, ng) fp32 master-grid scales, out (N,K) float64. */
int oq_dequant_f64(const uint8_t* codes, int N, int K, const float* scales, int ng,
                   int G, int c, int r, double* out) {
    if ((int64_t)(K - 1) / G >= ng && K > 0) return OQ_BAD_ARGS;
    const int64_t step = 1 << (c - r);
    const int64_t zr = 1 << (r - 1);
    for (int i = 0; i < N; i++)
        for (int j = 0; j < K; j++) {
            int q = codes[(size_t)i * K + j];
            if (q > (1 << r) - 1) return OQ_CODE_RANGE; /* grid.py:135-136 */
            double s = (double)scales[(size_t)i * ng + j / G];
            out[(size_t)i * K + j] = s * (double)(step * ((int64_t)q - zr));
        }
    return OQ_OK;
}

/* matmul.py:64-69 (PackedLayer.dense_f32): (float32(code) - float32(z)) *
 * scales_eff[:, col // G], one float32 rounding.  scales_eff are the child's
 * effective scales (slicing.py:127). */
void oq_dense_f32(const uint8_t* codes, int N, int K, const float* scales_eff, int ng,
                  int G, int r, float* W) {
    const float z = (float)(1 << (r - 1));
    for (int i = 0; i < N; i++)
        for (int j = 0; j < K; j++) {
            float q = (float)codes[(size_t)i * K + j];
            W[(size_t)i * K + j] = (q - z) * scales_eff[(size_t)i * ng + j / G];
        }
}

/* matmul.py:85-92 (matmul_ref): Y = 0; for k ascending:
 * Y += X[:, k][:, None] * Wd[:, k][None, :]  -- float32 product, then
 * float32 add, in that order (no FMA). */
void oq_matmul_ref(const float* X, int B, int K, const float* W, int N, float* Y) {
    for (int b = 0; b < B; b++)
        for (int n = 0; n < N; n++) Y[(size_t)b * N + n] = 0.0f;
    for (int k = 0; k < K; k++)
        for (int b = 0; b < B; b++) {
            const float x = X[(size_t)b * K + k];
            float* yb = Y + (size_t)b * N;
            for (int n = 0; n < N; n++) {
                float p = x * W[(size_t)n * K + k];
                yb[n] = yb[n] + p;
            }
        }
}

/* Dense float32 GEMV/GEMM, one thread: the reference bench's baseline
 * `X @ Wd.T` under threadpool_limits(1) (matmul.py:164-165).  Row-dot order
 * (BLAS-like); used only as the CPU timing baseline for r in {6, 8}, which
 * have no packed kernel in the reference (matmul.py:55-56). */
void oq_dense_gemm_f32(const float* X, int B, int K, const float* W, int N, float* Y) {
    for (int b = 0; b < B; b++) {
        const float* xb = X + (size_t)b * K;
        for (int n = 0; n < N; n++) {
            const float* wn = W + (size_t)n * K;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f, a5 = 0.f, a6 = 0.f, a7 = 0.f;
            int k = 0;
            for (; k + 8 <= K; k += 8) {
                a0 += xb[k] * wn[k];         a1 += xb[k + 1] * wn[k + 1];
                a2 += xb[k + 2] * wn[k + 2]; a3 += xb[k + 3] * wn[k + 3];
                a4 += xb[k + 4] * wn[k + 4]; a5 += xb[k + 5] * wn[k + 5];
                a6 += xb[k + 6] * wn[k + 6]; a7 += xb[k + 7] * wn[k + 7];
            }
            for (; k < K; k++) a0 += xb[k] * wn[k];
            Y[(size_t)b * N + n] = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
        }
    }
}

/* packing.py:81-110 (pack, canonical layout): columns zero-padded to a
 * multiple of 32 (packing.py:34-35, :91-93); per 32-weight unit a uint64
 * base word with code bits 0..1 of weight i at [2i, 2i+1] (packing.py:96),
 * a uint32 plane for bit 2 (bits >= 3, :98-100) and for bit 3 (bits == 4,
 * :101-103).  Returns OQ_CODE_RANGE on overflow (packing.py:88-89). */
int oq_pack_child(const uint8_t* codes, int N, int K, int bits,
                  uint64_t* base, uint32_t* b2, uint32_t* b3) {
    if (bits < 2 || bits > 4) return OQ_BAD_ARGS;
    const int nu = (K + 31) / 32;
    for (int64_t i = 0; i < (int64_t)N * K; i++)
        if (codes[i] >= (1 << bits)) return OQ_CODE_RANGE;
    for (int i = 0; i < N; i++)
        for (int u = 0; u < nu; u++) {
            uint64_t w = 0;
            uint32_t p2 = 0, p3 = 0;
            for (int l = 0; l < 32; l++) {
                int col = u * 32 + l;
                int q = col < K ? codes[(size_t)i * K + col] : 0;
                w |= (uint64_t)(q & 3) << (2 * l);
                p2 |= (uint32_t)((q >> 2) & 1) << l;
                p3 |= (uint32_t)((q >> 3) & 1) << l;
            }
            base[(size_t)i * nu + u] = w;
            if (bits >= 3) b2[(size_t)i * nu + u] = p2;
            if (bits == 4) b3[(size_t)i * nu + u] = p3;
        }
    return OQ_OK;
}

/* packing.py:113-126 (unpack): inverse of oq_pack_child, logical shape. */
void oq_unpack_child(const uint64_t* base, const uint32_t* b2, const uint32_t* b3,
                     int N, int K, uint8_t* codes) {
    const int nu = (K + 31) / 32;
    for (int i = 0; i < N; i++)
        for (int col = 0; col < K; col++) {
            int u = col / 32, l = col % 32;
            int q = (int)((base[(size_t)i * nu + u] >> (2 * l)) & 3u);
            if (b2) q |= (int)((b2[(size_t)i * nu + u] >> l) & 1u) << 2;
            if (b3) q |= (int)((b3[(size_t)i * nu + u] >> l) & 1u) << 3;
            codes[(size_t)i * K + col] = (uint8_t)q;
        }
}

/* Composite used by tests/bench: parent codes (N,K) at c bits + master-grid
 * scales (N, ng) -> r-bit child -> dense_f32 -> matmul_ref.  This is the
 * chain slice_layer (slicing.py:122-135) -> PackedLayer.from_sliced
 * (matmul.py:53-62; pack/unpack are lossless, packing.py:113-126) ->
 * matmul_ref (matmul.py:85-92); for r in {6, 8}, which PackedLayer rejects
 * (matmul.py:55-56), it is the same formula applied directly. */
int oq_parent_matmul_ref(const uint8_t* parent, int N, int K, const float* scales, int ng,
                         int G, int c, int r, const float* X, int B,
                         uint8_t* child_scratch, float* scale_scratch, float* W_scratch,
                         float* Y) {
    int st = oq_slice(parent, (int64_t)N * K, c, r, 0, child_scratch);
    if (st) return st;
    oq_scale_eff(scales, (int64_t)N * ng, c, r, scale_scratch);
    oq_dense_f32(child_scratch, N, K, scale_scratch, ng, G, r, W_scratch);
    oq_matmul_ref(X, B, K, W_scratch, N, Y);
    return OQ_OK;
}
