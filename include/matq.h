/* matq.h -- C ABI of libmatq.so, the B200 (sm_100a) sliced weight-only linear.
 *
 * This is the drop-in boundary for the reference's native layer.  The
 * reference binds its C kernels through Cython
 * (pkg/src/nestquant/kernels/_core.pyx:8-16 -> packed_kernels.h:17-30);
 * libmatq exports the equivalents below, plain pointers and sizes only.
 * INTEGRATION.md shows the Cython / ctypes stubs a maintainer adds.
 *
 * Conventions
 *   - Every pointer argument except the host-side query functions is a
 *     DEVICE pointer (cudaMalloc / torch CUDA tensor storage), caller-owned;
 *     libmatq never allocates or frees (as the reference C core never does,
 *     _core.pyx:42-45 allocates on the Python side).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Hot-path calls (mq_gemv, mq_pack_blob,
 *     mq_slice, mq_dequant, mq_materialize_child) are asynchronous, do no
 *     host synchronisation and no allocation, and are CUDA-graph capturable.
 *     The format helpers that validate data (mq_slice_elementwise,
 *     mq_dequant_f64, mq_pack_ref_layout) synchronise `stream` to report
 *     MQ_ERR_CODE_RANGE, as the reference validates synchronously.
 *   - Return value: MQ_OK or an MQ_ERR_* status; mq_last_error() gives a
 *     thread-local message (replaces the reference's Python-side exception
 *     texts, matmul.py:106-109, slicing.py:22-28, which the Python layer
 *     keeps verbatim).
 *
 * Device layout: a "blob" of uint32 blocks, one per (16-row
 * tile rt, 256-column step st), each = [scale block][plane 0 slab]...[plane
 * P-1 slab]; a slab is 32 lanes x 4 words = 512 B, plane 0 = code MSB, and the
 * scale block holds the fp32 group scales of the step (spg = 256/G groups x 16
 * rows for G in {32,64,128}; 1 group for G a multiple of 256; none otherwise).
 * A parent has P = nbits planes (8 for the int8 parent); an r-bit child
 * ("mode C") has P = r.  Slice r of a parent reads the first scale block +
 * (r+1) slabs of every block -- one contiguous bulk copy per step.
 * Np = ceil16(N), Kp = ceil256(K).  For G != 128 a tiled scale array
 * tscales fp32[Np/16][ceil(Kp/G)][16] accompanies the blob.
 */
#ifndef MATQ_H
#define MATQ_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MQ_API __attribute__((visibility("default")))
#else
#define MQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MQ_OK 0
#define MQ_ERR_INVALID 1    /* bad shape / bit-width / group size / pointer      */
#define MQ_ERR_CODE_RANGE 2 /* a code exceeds its bit-width                      */
#define MQ_ERR_WORKSPACE 3  /* workspace missing or smaller than required        */
#define MQ_ERR_CUDA 4       /* CUDA runtime error (see mq_last_error)            */

/* mq_gemv flags */
#define MQ_CHILD 1 /* informational: mode C is implied by nplanes == r */
#define MQ_X_F32 2 /* X is fp32 [B][ldx] (split on device into bf16 hi + lo terms); else bf16 */
#define MQ_Y_F32 4 /* Y is fp32 [B][ldy]; else bf16 */
#define MQ_PDL 8   /* programmatic dependent launch (overlap with the previous kernel) */

/* Capability query; replaces nq_simd_kind (packed_kernels.h:29-30,
 * packed_kernels.c:27).  Returns 100 for the sm_100a build. */
MQ_API int mq_arch(void);
MQ_API const char* mq_version(void);
MQ_API const char* mq_last_error(void);

/* Layout sizes (host-side, no CUDA calls). */
MQ_API int mq_layout_dims(int N, int K, int G, int* Np, int* Kp, int* ngp);
MQ_API size_t mq_blob_bytes(int N, int K, int G, int nplanes);
MQ_API size_t mq_tscales_bytes(int N, int K, int G);

/* K1: codes (N, K) uint8 with `nbits` significant bits (8 for the int8
 * parent, r for a child) + group scales (N, ceil(K/G)) fp32 row-major
 * (QuantGrid.scales, grid.py:75) -> blob (+ tscales, required when
 * G != 128).  Replaces the reference's child packer pack() (packing.py:81-110)
 * and its raw-byte parent storage (checkpoint.py:66-75) with one device
 * layout. */
MQ_API int mq_pack_blob(const uint8_t* codes, long long ldc, int N, int K, int nbits,
                        const float* scales, int G, uint32_t* blob, float* tscales, void* stream);

/* K2a: r-bit sliced codes (N, K) uint8 from a blob of `nplanes` planes, with
 * the bitsliced slice the GEMV uses (nplanes == r: the blob is a child).
 * Replaces slice_to_code over a layer (slicing.py:51-54, slice_layer
 * :158-171). */
MQ_API int mq_slice(const uint32_t* blob, int N, int K, int G, int nplanes, int r,
                    uint8_t* codes_out, long long ldo, void* stream);

/* K2b: decode through the exact GEMV register path.  vals_out (optional):
 * int8 s - 2^(r-1); w_out (optional): fp32 (s - z) * scale * out_scale, i.e.
 * PackedLayer.dense_f32 (matmul.py:64-69) when out_scale = 2^(c-r). */
MQ_API int mq_dequant(const uint32_t* blob, const float* tscales, int N, int K, int G, int nplanes,
                      int r, float out_scale, int8_t* vals_out, float* w_out, long long ldw,
                      void* stream);

/* K2c: materialise an r-plane child (mode C) from an 8-plane parent blob;
 * the child keeps the parent's master scales (use out_scale = 2^(8-r)). */
MQ_API int mq_materialize_child(const uint32_t* blob, int N, int K, int G, int r, uint32_t* child,
                                void* stream);

/* K3: Y = X @ dequant(slice_r(blob)).T, fp32 accumulation.
 * Replaces _core.packed_matmul (_core.pyx:24-64) -> nq_group_lane_sums /
 * nq_gemv / nq_gemm (packed_kernels.h:17-27), for r in {2,3,4,6,8} and
 * 1 <= B <= 32 (B <= 16 with MQ_X_F32).  X (B, K) with row stride ldx,
 * Y (B, N) with row stride ldy.  out_scale multiplies the tiled scales
 * (2^(c-r) for a parent slice, exact; 1.0 for a child with effective scales).
 * G must be a multiple of 32.  `workspace` must hold
 * mq_gemv_workspace_bytes(N, K, B, flags) bytes (0 when the launch needs no
 * cross-CTA split-K) and be zero-filled once at allocation: its first 64 KiB
 * are split-K tickets that every call leaves at zero, so one workspace (sized
 * for the largest layer) serves any sequence of GEMVs on one stream. */
MQ_API size_t mq_gemv_workspace_bytes(int N, int K, int B, int flags);
MQ_API int mq_gemv(const uint32_t* blob, const float* tscales, const void* X, int ldx, void* Y,
                   int ldy, int B, int N, int K, int G, int nplanes, int r, float out_scale,
                   int flags, void* workspace, size_t workspace_bytes, void* stream);

/* K4: the same product for prefill batches (any B, normally B > 32), on the
 * tcgen05 tensor cores: the decode warps slice + dequantise the blob into
 * shared memory as bf16 scale * (s - 2^(r-1)) and tcgen05.mma accumulates in
 * fp32 (TMEM).  X is bf16 (B, K), 16-byte aligned, ldx % 8 == 0; Y bf16 or
 * fp32 (MQ_Y_F32).  G must be 128.  `workspace` (zero-filled once, shared
 * with mq_gemv: same ticket convention) must hold
 * mq_gemm_workspace_bytes(N, K, B, flags) bytes -- nonzero only when the
 * tiles cannot fill the GPU and K is split across CTAs (deterministic
 * in-order reduction).  It does not take r: past 256 tokens the tiling may
 * depend on r (256- or 512-token tiles), so it returns the larger need.  Replaces the reference's blocked batch path nq_gemm
 * (packed_kernels.h:25-27) as driven by _core.pyx:53-63 for batch >= 8. */
MQ_API size_t mq_gemm_workspace_bytes(int N, int K, int B, int flags);
MQ_API int mq_gemm(const uint32_t* blob, const void* X, int ldx, void* Y, int ldy, int B, int N,
                   int K, int G, int nplanes, int r, float out_scale, int flags, void* workspace,
                   size_t workspace_bytes, void* stream);

/* K3S: a whole decode step -- every sliced linear of a model, in dependency
 * order (layer i+1 reads layer i's output) -- as ONE persistent cooperative
 * kernel (one CTA per SM).  Replaces a per-layer loop of mq_gemv calls (and
 * the reference's per-layer packed_matmul calls); each layer's weight ring
 * keeps streaming across layer boundaries while the previous layer drains.
 * G = 128, bf16 X/Y, 1 <= B <= 16.  r > 0: every layer sliced to r.  r = 0:
 * each layer's own r (mq_stack_layer.r; an EvoPress configuration), parents
 * only (nplanes = 8) -- one kernel dispatching per layer on its width.
 *   1. mq_stack_plan: host-only; fills a host plan (mq_stack_plan_bytes()) and
 *      a host layer table (mq_stack_table_bytes(n)) and returns the workspace
 *      size.  Copy the table to device memory (any time before the run).
 *   2. mq_stack_run: launches one step (async, graph-capturable).  The
 *      workspace must be zero-filled ONCE; its completion counters only grow,
 *      so steps replay without resets. */
typedef struct mq_stack_layer {
    const uint32_t* blob; /* P8 blob (parent: nplanes planes) */
    const void* X;        /* bf16 (B, K), row stride ldx, 16-byte aligned */
    void* Y;              /* bf16 (B, N), row stride ldy */
    int ldx, ldy, N, K;
    float out_scale;      /* 2^(c - r) for a parent slice */
    int r;                /* this layer's bits when mq_stack_plan's r = 0; else ignored */
    /* activation prologue fused into the layer's staging (0 = none):
     *   MQ_XOP_ADD_RMSNORM: R <- bf16(R + X); X' = bf16(R * rsqrt(mean(R^2) + eps) * norm_w), R the
     *     residual stream (res_in, or NULL: the residual the previous ADD_RMSNORM layer of this
     *     stack kept); CTA 0 writes the updated R to res_out when non-NULL;
     *   MQ_XOP_SILU_MUL: X' = bf16(bf16(silu(X[:, :K])) * X[:, K:2K]) (X is 2K wide).
     * The row-wise math of mq_add_rmsnorm / mq_silu_mul; an add-RMSNorm layer runs as one K chunk. */
    int xop;
    const void* res_in;   /* bf16 (B, K), row stride ldres */
    void* res_out;        /* bf16 (B, K), row stride ldres */
    const float* norm_w;  /* fp32 (K), 16-byte aligned */
    int ldres;
    float eps;
    /* output epilogue (0 = none):
     *   MQ_YOP_SILU_PAIRS: the layer's rows come in 16-row tiles of 8 gate rows followed by the
     *     8 matching up rows (a fused gate/up weight stored interleaved); Y is (B, N / 2):
     *     Y[:, 8t + i] = bf16(bf16(silu(bf16(g))) * bf16(u)), g / u = tile t's rows i / 8 + i --
     *     mq_silu_mul's math, done where the rows are finished (N % 16 == 0). */
    int yop;
} mq_stack_layer;
#define MQ_XOP_NONE 0
#define MQ_XOP_ADD_RMSNORM 1
#define MQ_XOP_SILU_MUL 2
#define MQ_YOP_NONE 0
#define MQ_YOP_SILU_PAIRS 1
MQ_API size_t mq_stack_plan_bytes(void);
MQ_API size_t mq_stack_table_bytes(int n_layers);
MQ_API int mq_stack_plan(const mq_stack_layer* layers, int n_layers, int B, int r, int nplanes,
                         void* plan_host, void* table_host, size_t* workspace_bytes);
MQ_API int mq_stack_run(const void* plan_host, const void* table_dev, void* workspace,
                        size_t workspace_bytes, void* stream);
/* The persistent kernel's step counter (64-bit; launch_ctr = launches * grid,
 * every layer's completion counter equal to it between steps).  set = 1 writes
 * *launches, set = 0 reads it (MQ_ERR_INVALID if the counters disagree).
 * Synchronous.  For tests and long-running servers that want to re-base it. */
MQ_API int mq_stack_epoch(const void* plan_host, void* workspace, size_t workspace_bytes,
                          unsigned long long* launches, int set, void* stream);

/* ---- format-layer helpers behind the drop-in Python API --------------- */

/* slice_code / slice_to_code (slicing.py:31-54) over n codes at master
 * bit-width c; err_dev: one device int of scratch.  Synchronises. */
MQ_API int mq_slice_elementwise(const uint8_t* q, long long n, int c, int r, int on_master,
                         uint8_t* out, int* err_dev, void* stream);

/* dequant (grid.py:128-149) in float64.  Synchronises. */
MQ_API int mq_dequant_f64(const uint8_t* codes, int N, int K, const float* scales, int ng, int G, int c,
                   int r, double* out, int* err_dev, void* stream);

/* dequant_value (grid.py:128-140): out[i] = scale[i] * (2^(c-r) * (q[i] - 2^(r-1)))
 * with a per-element float64 scale.  Synchronises. */
MQ_API int mq_dequant_value_f64(const uint8_t* q, const double* scale, long long n, int c, int r,
                                double* out, int* err_dev, void* stream);

/* matmul_ref (matmul.py:85-92), bit-exact float32 k-ascending. */
MQ_API int mq_matmul_ref(const float* X, int B, int K, const float* W, int N, float* Y, void* stream);

/* The reference's child bit-plane layout (packing.py:81-126).  Synchronises. */
MQ_API int mq_pack_ref_layout(const uint8_t* codes, int N, int K, int bits, uint64_t* base, uint32_t* b2,
                       uint32_t* b3, int* err_dev, void* stream);
MQ_API int mq_unpack_ref_layout(const uint64_t* base, const uint32_t* b2, const uint32_t* b3, int N, int K,
                         uint8_t* codes, void* stream);

/* ---- MatGPTQ quantiser searches, float64 ---------- *
 * A BitWidthSet (grid.py:27-66) is passed as host arrays targets[T]
 * (distinct, ascending, in [2, 8]; the last is the master width c) and
 * lams[T] (positive).  Matrices are row-major device float64 with a row
 * stride; scales are float32 (d_row, ngs) group scales.  Results are
 * bit-identical to the reference's numpy (same operation order, no FMA
 * contraction).  All three are asynchronous. */

/* select_codes (gptq.py:104-140): per weight, the master code minimising
 * sum_t lams[t] * (w - s * mv_t[q])^2; ties to the smallest code. */
MQ_API int mq_select_codes(const double* W, long long ldw, int d_row, int d_col, const float* scales,
                           int ngs, int G, const int* targets, const double* lams, int T, uint8_t* codes,
                           long long ldc, void* stream);

/* fit_grid (grid.py:160-212): the shrink search over alphas[steps] (device,
 * numpy.linspace(1, shrink_min, steps)) per (row, group) -> float32 scales
 * (d_row, ceil(d_col / G)). */
MQ_API int mq_fit_grid(const double* W, long long ldw, int d_row, int d_col, int G, const int* targets,
                       const double* lams, int T, const double* alphas, int steps, float* scales, void* stream);

/* rtn (grid.py:114-125): codes[i] = clip(round_half_away(w[i] / scale[i] +
 * 2^(c-1)), 0, 2^c - 1) as int64 over n broadcast elements (the caller
 * broadcasts w and scale); MQ_ERR_CODE_RANGE with "non-finite weight" when any
 * w is not finite.  Synchronises the stream (the error flag is read back). */
MQ_API int mq_rtn_f64(const double* w, const double* scale, long long n, int c, long long* codes, int* err_dev,
                      void* stream);
/* round_half_away (grid.py:108-111): nearest integer, halves away from zero,
 * float64 -> float64.  Asynchronous. */
MQ_API int mq_round_half_away_f64(const double* x, long long n, double* out, void* stream);

/* One column block [lo, hi) of quantize_layer's loop (gptq.py:203-222):
 * codes[:, lo:hi], the compensated snapshot comp[:, lo:hi], the scaled errors
 * err (d_row, hi - lo), and Wc's in-block rank-1 updates.  The caller applies
 * Wc[:, hi:] -= err @ chol[lo:hi, hi:] (a dgemm) before the next block. */
MQ_API int mq_gptq_block(double* Wc, long long ldw, int d_row, int d_col, int lo, int hi, const float* scales,
                         int ngs, int G, const double* chol, long long ldch, const int* targets,
                         const double* lams, int T, uint8_t* codes, long long ldc, double* comp,
                         long long ldcomp, double* err, long long lde, void* stream);

/* ---- full-model decode harness glue (llama.py), bf16 --
 * Not part of the sliced linear: the row-wise steps between a Llama block's
 * linears, fused so a block is 4 linears + 3 glue launches + attention.
 * mq_add_rmsnorm: x += delta (when delta is non-null; x is the bf16 residual
 *   stream), y = x * rsqrt(mean(x^2) + eps) * w (w float32), per row of h.
 * mq_rope_kv: rotary embedding (rotate-half, cos/sin bf16 of head_dim / 2) of
 *   the q and k heads of a fused qkv row; q -> (B, n_heads, head_dim); k and v
 *   written into (B, n_kv_heads, T, head_dim) caches at position pos.
 * mq_silu_mul: y = silu(g) * u for rows [g | u] of 2 * inter. */
MQ_API int mq_add_rmsnorm(void* x, const void* delta, const float* w, void* y, int B, int h, float eps,
                          void* stream);
MQ_API int mq_rope_kv(const void* qkv, const void* cosv, const void* sinv, void* q, void* kcache, void* vcache,
                      int B, int n_heads, int n_kv_heads, int head_dim, int T, int pos, void* stream);
/* mq_qknorm_rope_kv: mq_rope_kv with a per-head RMSNorm of q and k first
 *   (Qwen3's q_norm / k_norm weights, fp32 of head_dim; eps 1e-6). */
MQ_API int mq_qknorm_rope_kv(const void* qkv, const void* cosv, const void* sinv, void* q, void* kcache,
                             void* vcache, int B, int n_heads, int n_kv_heads, int head_dim, int T, int pos,
                             const float* q_norm, const float* k_norm, float eps, void* stream);
MQ_API int mq_silu_mul(const void* gu, void* y, int B, int inter, void* stream);
/* mq_attn_decode: single-query decode attention for the decoder harness, with the
 *   (optional q/k RMSNorm +) rotary step and the KV-cache write fused in: grid (n_heads, B);
 *   q head h attends over cache rows [0, pos) of kv head kv_of_q[h] plus its new k / v
 *   (written at pos by the first q head of each kv head); fp32 softmax (1/sqrt(head_dim));
 *   att (B, n_heads * head_dim) bf16.  head_dim 64 or 128, pos < 51200 (the scores live in
 *   shared memory). */
MQ_API int mq_attn_decode(const void* qkv, const void* cosv, const void* sinv, const float* q_norm,
                          const float* k_norm, float eps, void* kcache, void* vcache, const int* kv_of_q,
                          void* att, int B, int n_heads, int n_kv_heads, int head_dim, int T, int pos,
                          void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MATQ_H */
