// matq_abi.cu -- extern "C" entry points of libmatq.so (include/matq.h):
// argument validation, launch configuration, error reporting.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/matq.h"
#include "matq_gemv.cuh"
#include "matq_internal.h"
#include "matq_stack.cuh"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return MQ_OK;
    return fail(MQ_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool valid_r(int r) { return r == 2 || r == 3 || r == 4 || r == 6 || r == 8; }

int sm_count() {
    static int cached[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        cached[dev] = n;
    }
    return cached[dev];
}

struct GemvConfig {
    int NT, S, cs, grid, nwarps, stages;
    int slots;  // partial-sum slots per row tile (= S)
    size_t smem;
    int xs_stride, xs_bytes, xcopy_stride, cs_off;
    int pair, pair_units, pair_off;  // S == 2 on CTA pairs (DSMEM reduction)
};

constexpr size_t kXsMax = 48 * 1024;        // activations staged per CTA (chunked mode)
constexpr size_t kSmemFullSm = 220 * 1024;

int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

// Decomposition.  One CTA of `nwarps` independent warps per
// SM.  The cost of a configuration is the critical path in steps on the most
// loaded SM sub-partition (4 per SM, warp w on SMSP w % 4), since the decode
// is issue-bound per SMSP; a split tile adds a fixup (partials + ticket).
// K is cut into S chunks of cs steps, row tiles dealt warp-major; every tile
// of an S > 1 split needs the fixup.  (A stream-K assignment -- balanced
// contiguous per-warp ranges -- was measured and lost to the fixups; see
// DESIGN.md 4.)
GemvConfig choose_gemv_config(int N, int K, int Bx, int npl, bool g128, int r,
                              bool honour_overrides = true, int force_warps = 0) {
    GemvConfig c{};
    const int n_rt = mq::pad16(N) / 16, nsteps = mq::pad256(K) / 256;
    c.NT = Bx <= 8 ? 1 : (Bx <= 16 ? 2 : 4);
    const int ncopy = (g128 && r != 8 && c.NT == 1) ? mq::zp_ncopies(r) : 1;  // k_gemv's ZP rule
    // staging budget: fewer warps' rings at NT = 4 leave room for longer K chunks
    const size_t xs_max = c.NT >= 4 ? 96 * 1024 : (c.NT == 2 ? 64 * 1024 : kXsMax);
    // tuning overrides (scripts/sweep_gemv.py): MQ_GEMV_WARPS, MQ_GEMV_SPLIT, MQ_GEMV_STAGES,
    // MQ_GEMV_STREAM (0 = never, 1 = force when it fits)
    c.nwarps = force_warps ? force_warps
                           : std::max(4, std::min(mq::kMaxWarps, env_int("MQ_GEMV_WARPS", c.NT >= 4 ? 8 : 16)));
    c.nwarps &= ~3;
    const int force_s = honour_overrides ? env_int("MQ_GEMV_SPLIT", 0) : 0;
    const double fixup = 2.0;  // measured: a split-K tile costs ~2 steps (partials, ticket, reduction)
    // CTA pairs (clusters of 2) reduce S = 2 through DSMEM for ~nothing (MQ_GEMV_PAIR=0: off)
    const bool pair_ok = env_int("MQ_GEMV_PAIR", 1) != 0 && sm_count() % 2 == 0;
    const int sms = sm_count();
    double best = 1e30;
    for (int S_try = 1; S_try <= std::min(nsteps, 64); ++S_try) {
        if (force_s && S_try != std::min(force_s, nsteps)) continue;
        const int cs = mq::cdiv(nsteps, S_try);
        // a chunk count that would leave an empty chunk is never used: its
        // CTAs would not take a ticket and the tile's fixup would never run
        // (a forced MQ_GEMV_SPLIT is rounded to the effective chunk count)
        const int S = mq::cdiv(nsteps, cs);
        if (S != S_try && !force_s) continue;
        const size_t xs = (size_t)ncopy * Bx * (cs * 256 + 8) * 2;
        if (xs > xs_max && cs > 1) continue;
        int cpc = sms / S;
        if (cpc < 1) break;
        cpc = std::min(cpc, n_rt);  // at least one row tile per CTA
        const int rt_stride = cpc * c.nwarps;
        // most units on one SMSP: CTA 0, SMSP 0 (warps 0, 4, 8, ... take the
        // lowest tile indices, and a warp's unit count is non-increasing in it)
        int max_units = 0;
        for (int w = 0; w < c.nwarps; w += 4) {
            const int first = w * cpc;
            if (first < n_rt) max_units += (n_rt - 1 - first) / rt_stride + 1;
        }
        const double fix = S == 1 ? 0.0 : (pair_ok && S == 2 ? 0.3 : fixup);
        const double cost = (double)max_units * (cs + fix);
        if (cost < best - 1e-9) {
            best = cost;
            c.S = S;
            c.cs = cs;
            c.grid = cpc * S;
        }
    }
    if (c.S == 0)  // overrides admitted no configuration: ignore them
        return choose_gemv_config(N, K, Bx, npl, g128, r, false, force_warps);
    c.slots = c.S;
    c.xs_stride = c.cs * 256 + 8;
    c.xcopy_stride = Bx * c.xs_stride;
    c.cs_off = (int)(((size_t)ncopy * c.xcopy_stride * 2 + 15) & ~(size_t)15);
    // zero-point constants whenever k_gemv folds the zero point (its ZP rule; r = 6
    // folds with a single activation copy, so this is not ncopy > 1)
    const bool zp = g128 && r != 8 && c.NT == 1;
    const size_t zc_bytes = zp ? (size_t)2 * c.cs * c.NT * 8 * 4 : 0;
    c.xs_bytes = (int)((c.cs_off + zc_bytes + 15) & ~(size_t)15);
    c.pair = pair_ok && c.S == 2 && c.grid % 2 == 0;
    if (c.pair) {
        const int rt_stride = (c.grid / c.S) * c.nwarps;
        c.pair_units = mq::cdiv(n_rt, rt_stride);
        c.pair_off = c.xs_bytes;
        const size_t pb = (((size_t)8 * mq::kMaxWarps * c.pair_units + 15) & ~(size_t)15) +
                          (size_t)mq::kMaxWarps * c.pair_units * 32 * c.NT * 16;
        c.xs_bytes = (int)((c.pair_off + pb + 15) & ~(size_t)15);
    }
    const size_t stage = (size_t)npl * 512 + (g128 ? 128 : 0);
    const size_t fixed = (size_t)c.xs_bytes + mq::kMaxWarps * 8 * 8;
    int d = (int)((kSmemFullSm - std::min(fixed, kSmemFullSm)) / (c.nwarps * stage));
    c.stages = std::max(1, std::min(std::min(8, env_int("MQ_GEMV_STAGES", 4)), d));
    c.smem = fixed + (size_t)c.nwarps * c.stages * stage;
    return c;
}

// Workspace layout: [kTicketBytes of int tickets][fp32 partials].  The ticket
// region has a fixed size so that every GEMV sharing a workspace (any shape,
// any decomposition) finds its tickets where the previous one left them at 0.
constexpr size_t kTicketBytes = 64 * 1024;
constexpr int kMaxTickets = (int)(kTicketBytes / sizeof(int));

size_t gemv_ws_bytes(int N, const GemvConfig& c, int B) {
    if (c.slots <= 1) return 0;
    return kTicketBytes + (size_t)c.slots * B * mq::pad16(N) * sizeof(float);
}

// Configurations are pure functions of (shape, batch, path, overrides): cache them.
struct CfgKey {
    int N, K, Bx, npl, g128, r, w, s, st, sk;
    bool operator<(const CfgKey& o) const {
        return std::tie(N, K, Bx, npl, g128, r, w, s, st, sk) <
               std::tie(o.N, o.K, o.Bx, o.npl, o.g128, o.r, o.w, o.s, o.st, o.sk);
    }
};
GemvConfig cached_config(int N, int K, int Bx, int npl, bool g128, int r) {
    static std::mutex mu;
    static std::map<CfgKey, GemvConfig> cache;
    const CfgKey key{N, K, Bx, npl, (int)g128, r, env_int("MQ_GEMV_WARPS", 0), env_int("MQ_GEMV_SPLIT", 0),
                     env_int("MQ_GEMV_STAGES", 0), env_int("MQ_GEMV_PAIR", 1)};
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    const GemvConfig c = choose_gemv_config(N, K, Bx, npl, g128, r);
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = c;
    return c;
}

#ifdef MQ_GEMV_TIMING
unsigned long long* dbg_buffer() {
    static unsigned long long* buf = nullptr;
    if (!buf) {
        const size_t bytes = sizeof(unsigned long long) * (size_t)mq::kTsSlots * mq::kTsCtas * mq::kTsEvents;
        if (cudaMalloc(&buf, bytes) == cudaSuccess) cudaMemset(buf, 0, bytes);
    }
    return buf;
}
#endif

mq::GemvLaunchFn gemv_launcher(int r) {
    switch (r) {
        case 2: return mq::launch_gemv_r<2>;
        case 3: return mq::launch_gemv_r<3>;
        case 4: return mq::launch_gemv_r<4>;
        case 6: return mq::launch_gemv_r<6>;
        case 8: return mq::launch_gemv_r<8>;
    }
    return nullptr;
}

}  // namespace

extern "C" {

int mq_arch(void) { return 100; }

const char* mq_version(void) { return "matq 0.1.0 (sm_100a)"; }

#ifdef MQ_GEMV_TIMING
// Profiling builds only (scripts/phase_timing.py): phase timestamps of the last 64 K3 launches.
MQ_API int mq_debug_timestamps(unsigned long long* out, int n) {
    const size_t bytes = sizeof(unsigned long long) * (size_t)mq::kTsSlots * mq::kTsCtas * mq::kTsEvents;
    if ((size_t)n * sizeof(unsigned long long) < bytes) return MQ_ERR_INVALID;
    if (cudaMemcpy(out, dbg_buffer(), bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return MQ_ERR_CUDA;
    return MQ_OK;
}
MQ_API int mq_debug_gemm_timestamps(unsigned long long* out, int n) {
    if (n < 64 * 160 * 6) return MQ_ERR_INVALID;
    return cudaMemcpy(out, mq::gemm_dbg_buffer(), sizeof(unsigned long long) * 64 * 160 * 6,
                      cudaMemcpyDeviceToHost) == cudaSuccess ? MQ_OK : MQ_ERR_CUDA;
}
MQ_API int mq_debug_reset(void) {
    const size_t bytes = sizeof(unsigned long long) * (size_t)mq::kTsSlots * mq::kTsCtas * mq::kTsEvents;
    return cudaMemset(dbg_buffer(), 0, bytes) == cudaSuccess ? MQ_OK : MQ_ERR_CUDA;
}
#endif

const char* mq_last_error(void) { return g_err; }

int mq_layout_dims(int N, int K, int G, int* Np, int* Kp, int* ngp) {
    if (N < 1 || K < 1 || G < 1) return fail(MQ_ERR_INVALID, "bad layout dims N=%d K=%d G=%d", N, K, G);
    if (Np) *Np = mq::pad16(N);
    if (Kp) *Kp = mq::pad256(K);
    if (ngp) *ngp = mq::cdiv(mq::pad256(K), G);
    return MQ_OK;
}

size_t mq_blob_bytes(int N, int K, int G, int nplanes) {
    if (N < 1 || K < 1 || G < 1 || nplanes < 1 || nplanes > 8) return 0;
    return (size_t)mq::Layout::make(N, K, G, nplanes).total_words() * 4;
}

size_t mq_tscales_bytes(int N, int K, int G) {
    if (N < 1 || K < 1 || G < 1) return 0;
    return (size_t)mq::pad16(N) * mq::cdiv(mq::pad256(K), G) * sizeof(float);
}

static bool valid_group(int G) { return G >= 32 && G % 32 == 0; }

int mq_pack_blob(const uint8_t* codes, long long ldc, int N, int K, int nbits, const float* scales,
                 int G, uint32_t* blob, float* tscales, void* stream) {
    if (!codes || !blob || !scales) return fail(MQ_ERR_INVALID, "null pointer");
    if (N < 1 || K < 1 || ldc < K) return fail(MQ_ERR_INVALID, "bad shape N=%d K=%d ldc=%lld", N, K, ldc);
    if (nbits < 2 || nbits > 8) return fail(MQ_ERR_INVALID, "nbits must lie in [2, 8]");
    if (!valid_group(G)) return fail(MQ_ERR_INVALID, "group size must be a multiple of 32");
    if (G != 128 && !tscales) return fail(MQ_ERR_INVALID, "tscales required when G != 128");
    const mq::Layout L = mq::Layout::make(N, K, G, nbits);
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = mq::launch_pack_planes(codes, ldc, L, nbits, blob, s);
    if (e == cudaSuccess) e = mq::launch_pack_scales(scales, L, mq::cdiv(K, G), blob, tscales, s);
    return cuda_status(e, "mq_pack_blob");
}

static int check_slice(const uint32_t* blob, int N, int K, int G, int nplanes, int r) {
    if (!blob) return fail(MQ_ERR_INVALID, "null pointer");
    if (!valid_r(r)) return fail(MQ_ERR_INVALID, "unsupported bits");
    if (N < 1 || K < 1) return fail(MQ_ERR_INVALID, "bad shape");
    if (!valid_group(G)) return fail(MQ_ERR_INVALID, "group size must be a multiple of 32");
    if (nplanes < r || nplanes > 8) return fail(MQ_ERR_INVALID, "cannot slice %d bits out of %d", r, nplanes);
    if (nplanes != r && nplanes < r + 1) return fail(MQ_ERR_INVALID, "need %d planes", r + 1);
    return MQ_OK;
}

int mq_slice(const uint32_t* blob, int N, int K, int G, int nplanes, int r, uint8_t* codes_out,
             long long ldo, void* stream) {
    int st = check_slice(blob, N, K, G, nplanes, r);
    if (st) return st;
    if (!codes_out || ldo < K) return fail(MQ_ERR_INVALID, "bad output");
    const mq::Layout L = mq::Layout::make(N, K, G, nplanes);
    return cuda_status(mq::launch_slice_codes(r, nplanes == r, blob, L, codes_out, ldo,
                                              (cudaStream_t)stream),
                       "mq_slice");
}

int mq_dequant(const uint32_t* blob, const float* tscales, int N, int K, int G, int nplanes, int r,
               float out_scale, int8_t* vals_out, float* w_out, long long ldw, void* stream) {
    int st = check_slice(blob, N, K, G, nplanes, r);
    if (st) return st;
    if (!vals_out && !w_out) return fail(MQ_ERR_INVALID, "null pointer");
    const mq::Layout L = mq::Layout::make(N, K, G, nplanes);
    if (w_out && L.spg == 0 && !tscales) return fail(MQ_ERR_INVALID, "w_out needs tscales");
    if (ldw < K) return fail(MQ_ERR_INVALID, "bad shape");
    return cuda_status(mq::launch_decode_dense(r, nplanes == r, blob, tscales, L, out_scale, vals_out,
                                               w_out, ldw, (cudaStream_t)stream),
                       "mq_dequant");
}

int mq_materialize_child(const uint32_t* blob, int N, int K, int G, int r, uint32_t* child,
                         void* stream) {
    int st = check_slice(blob, N, K, G, 8, r);
    if (st) return st;
    if (!child) return fail(MQ_ERR_INVALID, "null pointer");
    if (r == 8) return fail(MQ_ERR_INVALID, "an 8-bit child is the parent");
    const mq::Layout L = mq::Layout::make(N, K, G, 8);
    return cuda_status(mq::launch_materialize_child(r, blob, L, child, (cudaStream_t)stream),
                       "mq_materialize_child");
}

size_t mq_gemv_workspace_bytes(int N, int K, int B, int flags) {
    if (N < 1 || K < 1 || B < 1) return 0;
    const int Bx = (flags & MQ_X_F32) ? 2 * B : B;
    if (Bx > 32) return 0;
    // the largest requirement over every bit-width / mode / group-size path
    size_t need = 0;
    for (int r : {2, 3, 4, 6, 8})
        for (int npl : {r, std::min(8, r + 1)})
            for (bool g128 : {true, false})
                need = std::max(need, gemv_ws_bytes(N, cached_config(N, K, Bx, npl, g128, r), B));
    return need;
}

int mq_gemv(const uint32_t* blob, const float* tscales, const void* X, int ldx, void* Y, int ldy,
            int B, int N, int K, int G, int nplanes, int r, float out_scale, int flags,
            void* workspace, size_t workspace_bytes, void* stream) {
    if (!blob || !X || !Y) return fail(MQ_ERR_INVALID, "null pointer");
    if (G != 128 && !tscales) return fail(MQ_ERR_INVALID, "tscales required when G != 128");
    if (nplanes < r || nplanes > 8 || (nplanes != r && nplanes < r + 1))
        return fail(MQ_ERR_INVALID, "cannot slice %d bits out of %d planes", r, nplanes);
    if (!valid_r(r)) return fail(MQ_ERR_INVALID, "unsupported bits");
    if (G < 32 || G % 32 != 0) return fail(MQ_ERR_INVALID, "group size must be a multiple of 32");
    if (N < 1 || K < 1 || B < 1) return fail(MQ_ERR_INVALID, "bad shape B=%d N=%d K=%d", B, N, K);
    if (ldx < K || ldy < N) return fail(MQ_ERR_INVALID, "bad leading dimension");
    const bool xf32 = flags & MQ_X_F32;
    const int Bx = xf32 ? 2 * B : B;
    if (Bx > 32) return fail(MQ_ERR_INVALID, "batch %d above the GEMV limit (32 rows, 16 with fp32 X)", B);

    const bool child_mode = nplanes == r;
    const int npl = (child_mode || r == 8) ? r : r + 1;
    const GemvConfig c = cached_config(N, K, Bx, npl, G == 128, r);
    const size_t need = gemv_ws_bytes(N, c, B);
    if (need > workspace_bytes || (need && !workspace))
        return fail(MQ_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);

    const mq::Layout L = mq::Layout::make(N, K, G, nplanes);
    mq::GemvParams p{};
    p.blob = blob;
    p.step_words = L.step_words;
    p.sb_words = 16 * L.spg;
    p.tscales = tscales;
    p.X = X;
    p.Y = Y;
    const int n_rt = mq::pad16(N) / 16;
    if (need) {
        if (n_rt > kMaxTickets) return fail(MQ_ERR_INVALID, "N=%d too large for split-K", N);
        p.tickets = reinterpret_cast<int*>(workspace);
        p.ws = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + kTicketBytes);
    }
    p.out_scale = out_scale;
    p.ldx = ldx;
    p.ldy = ldy;
    p.B = B;
    p.Bx = Bx;
    p.N = N;
    p.Np = mq::pad16(N);
    p.K = K;
    p.Kp = mq::pad256(K);
    p.G = G;
    p.ngp = mq::cdiv(p.Kp, G);
    p.nsteps = p.Kp / 256;
    p.n_rt = n_rt;
    p.S = c.S;
    p.cs = c.cs;
    p.ctas_per_chunk = c.grid / c.S;
    p.x_f32 = xf32 ? 1 : 0;
    p.y_f32 = (flags & MQ_Y_F32) ? 1 : 0;
    p.xs_stride = c.xs_stride;
    p.xcopy_stride = c.xcopy_stride;
    p.cs_off = c.cs_off;
    p.xs_bytes = c.xs_bytes;
    p.stages = c.stages;
    p.pair = c.pair;
    p.pair_off = c.pair_off;
    p.pair_units = c.pair_units;
#ifdef MQ_GEMV_TIMING
    static int dbg_ctr = 0;
    p.dbg_slot = dbg_ctr++ % mq::kTsSlots;
    p.dbg_ts = dbg_buffer();
#endif
    const dim3 grid(c.grid, 1, 1), block(32 * c.nwarps, 1, 1);
    const int gs = (G == 128) ? 128 : 0;
    const cudaError_t e = gemv_launcher(r)(p, c.NT, child_mode, gs, grid, block, c.smem,
                                           (cudaStream_t)stream, (flags & MQ_PDL) != 0);
    return cuda_status(e, "mq_gemv");
}

size_t mq_gemm_workspace_bytes(int N, int K, int B, int flags) {
    (void)flags;
    if (N < 1 || K < 1 || B < 1) return 0;
    // r is not an argument: the larger of the 256- and 512-token tilings' needs
    return std::max(mq::gemm_ws_bytes(mq::choose_gemm_config(N, K, B, sm_count(), 4)),
                    mq::gemm_ws_bytes(mq::choose_gemm_config(N, K, B, sm_count(), 8)));
}

int mq_gemm(const uint32_t* blob, const void* X, int ldx, void* Y, int ldy, int B, int N, int K,
            int G, int nplanes, int r, float out_scale, int flags, void* workspace,
            size_t workspace_bytes, void* stream) {
    if (!blob || !X || !Y) return fail(MQ_ERR_INVALID, "null pointer");
    if (nplanes < r || nplanes > 8 || (nplanes != r && nplanes < r + 1))
        return fail(MQ_ERR_INVALID, "cannot slice %d bits out of %d planes", r, nplanes);
    if (!valid_r(r)) return fail(MQ_ERR_INVALID, "unsupported bits");
    if (G != 128) return fail(MQ_ERR_INVALID, "mq_gemm needs group size 128 (got %d)", G);
    if (N < 1 || K < 1 || B < 1) return fail(MQ_ERR_INVALID, "bad shape B=%d N=%d K=%d", B, N, K);
    if (ldx < K || ldy < N) return fail(MQ_ERR_INVALID, "bad leading dimension");
    if (flags & MQ_X_F32) return fail(MQ_ERR_INVALID, "mq_gemm takes bf16 activations");
    if ((ldx & 7) || (reinterpret_cast<uintptr_t>(X) & 15))
        return fail(MQ_ERR_INVALID, "activations must be 16-byte aligned with ldx %% 8 == 0");
    const mq::GemmConfig c = mq::choose_gemm_config(N, K, B, sm_count(), r);
    const size_t need = mq::gemm_ws_bytes(c);
    if (need > workspace_bytes || (need && !workspace))
        return fail(MQ_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);
    if (need && c.n_tiles > (int)(mq::kGemmTicketBytes / sizeof(int)))
        return fail(MQ_ERR_INVALID, "too many tiles for split-K");
    const mq::Layout L = mq::Layout::make(N, K, G, nplanes);
    const char* why = "";
    const cudaError_t e = mq::launch_gemm(blob, L, X, ldx, Y, ldy, B, r, nplanes == r, out_scale,
                                          (flags & MQ_Y_F32) != 0, c, workspace, (cudaStream_t)stream,
                                          (flags & MQ_PDL) != 0, &why);
    if (e != cudaSuccess && *why) return fail(MQ_ERR_CUDA, "mq_gemm: %s", why);
    return cuda_status(e, "mq_gemm");
}

// ---- K3S: the whole decode step as one persistent kernel ---------------------
namespace {
struct StackPlanHost {  // the opaque host plan (mq_stack_plan_bytes)
    mq::StackParams p;
    int r, nplanes, nt, grid;
    size_t smem;
    size_t ws_bytes;
    size_t ll_bytes;
    size_t tk_bytes;
};
// K3S per-layer decomposition: K chunks S (activation staging bounded by
// kXsMax), the chunk's row tiles split contiguously over cpc = sms / S CTAs,
// and each CTA's (tile, step) pairs split evenly over its 16 warps.  Cost =
// the busiest SMSP's steps (4 warps share one) + a split-K fixup allowance.
struct StackCfg {
    int S, cs, cpc;
};
// pair: CTA pairs (clusters of 2) reduce S = 2 through DSMEM for ~free; S > 2
// still goes through the global workspace and tickets (~2 us of tail: partial
// stores, an acq_rel ticket and the last chunk's reloads).
StackCfg choose_stack_config(int N, int K, int B, int ncopy, int sms, size_t kXsMaxStack, bool pair,
                             bool one_chunk = false) {
    const int n_rt = mq::pad16(N) / 16, nsteps = mq::pad256(K) / 256;
    StackCfg best_c{nsteps, 1, std::max(1, std::min(sms / nsteps, n_rt))};
    double best = 1e30;
    for (int S_try = 1; S_try <= nsteps; ++S_try) {
        const int cs = mq::cdiv(nsteps, S_try);
        const int S = mq::cdiv(nsteps, cs);
        if (S != S_try) continue;
        const size_t xs = (size_t)ncopy * B * (cs * 256 + 8) * 2;
        if (xs > kXsMaxStack && cs > 1) continue;
        if (one_chunk && S_try > 1) break;  // a fused row-wise prologue needs the whole row
        const int cpc = std::min(sms / S, n_rt);
        if (cpc < 1) break;
        // busiest CTA: S = 1 splits the layer's (tile, step) pairs stream-K style
        // (every CTA within one step of the mean); S > 1 deals whole tiles per chunk
        const int work = S == 1 ? mq::cdiv((long long)n_rt * nsteps, sms) : mq::cdiv(n_rt, cpc) * cs;
        const double per_warp = (double)mq::cdiv(work, mq::kStackWarps);
        const double fix = S == 1 ? 0.0 : (pair && S == 2 ? 0.5 : (pair ? 6.0 : 3.0));
        const double cost = 4.0 * per_warp + fix + (work % mq::kStackWarps ? 0.5 : 0.0);
        if (cost < best - 1e-9) {
            best = cost;
            best_c = StackCfg{S, cs, cpc};
        }
    }
    return best_c;
}

// workspace: [tickets (per layer, self-resetting)][done counters n + launch counter][LL words][partials]
size_t stack_ws_layout(int n_layers, size_t ll_bytes, size_t partial_bytes, size_t* off_done, size_t* off_ll,
                       size_t* off_partials, size_t ticket_bytes) {
    *off_done = (ticket_bytes + 255) & ~(size_t)255;
    *off_ll = *off_done + (((size_t)(n_layers + 1) * 8 + 255) & ~(size_t)255);
    *off_partials = *off_ll + ((ll_bytes + 255) & ~(size_t)255);
    return *off_partials + partial_bytes;
}

// Which earlier layer produces layer i's X?  The latest layer j whose Y overlaps
// X decides: X must lie entirely inside Y_j (same row stride, even element
// offset) -- then layer i polls j's LL words -- else the stack cannot order the
// two (-2).  -1: no earlier layer writes X (activations from outside the step).
int stack_out_width(const mq_stack_layer& o) { return o.yop == MQ_YOP_SILU_PAIRS ? o.N / 2 : o.N; }
int stack_x_producer(const mq_stack_layer* layers, int i, int B, size_t* elem_off) {
    const mq_stack_layer& in = layers[i];
    const int xw = in.xop == MQ_XOP_SILU_MUL ? 2 * in.K : in.K;  // columns of X the layer reads
    auto lo = [](const void* p) { return reinterpret_cast<uintptr_t>(p); };
    const uintptr_t x0 = lo(in.X), x1 = x0 + 2 * ((size_t)(B - 1) * in.ldx + xw);
    for (int j = i - 1; j >= 0; --j) {
        const mq_stack_layer& o = layers[j];
        const int on = stack_out_width(o);
        const uintptr_t y0 = lo(o.Y), y1 = y0 + 2 * ((size_t)(B - 1) * o.ldy + on);
        if (x1 <= y0 || y1 <= x0) continue;  // no overlap: look further back
        const size_t e = (x0 - y0) / 2;  // X's first element inside Y (row 0: both have B rows)
        const bool inside = o.ldy == in.ldx && x0 >= y0 && (x0 - y0) % 4 == 0 && e + (size_t)xw <= (size_t)on;
        *elem_off = e;
        return inside ? j : -2;
    }
    return -1;
}
bool stack_overlap(const void* a, int lda, int na, const void* b, int ldb, int nb, int B) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), a1 = a0 + 2 * ((size_t)(B - 1) * lda + na);
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(b), b1 = b0 + 2 * ((size_t)(B - 1) * ldb + nb);
    return !(a1 <= b0 || b1 <= a0);
}
}  // namespace

#ifdef MQ_GEMV_TIMING
static unsigned long long* g_stack_dbg = nullptr;
MQ_API int mq_debug_stack_timestamps(unsigned long long* out, int n) {
    const size_t bytes = sizeof(unsigned long long) * (256 * 148 * 8 + 256 * 16 * 4);
    if (!g_stack_dbg || (size_t)n * 8 < bytes) return MQ_ERR_INVALID;
    return cudaMemcpy(out, g_stack_dbg, bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? MQ_OK : MQ_ERR_CUDA;
}
#endif

size_t mq_stack_plan_bytes(void) { return sizeof(StackPlanHost); }
size_t mq_stack_table_bytes(int n_layers) { return n_layers < 0 ? 0 : sizeof(mq::StackLayer) * (size_t)n_layers; }

static int stack_plan_impl(const mq_stack_layer* layers, int n_layers, int B, int r, int nplanes,
                           void* plan_host, void* table_host, size_t* workspace_bytes, bool pair) {
    if (!layers || !plan_host || !table_host || !workspace_bytes || n_layers < 1)
        return fail(MQ_ERR_INVALID, "null pointer or empty stack");
    if (r != 0 && !valid_r(r)) return fail(MQ_ERR_INVALID, "unsupported bits");
    if (r == 0 && nplanes != 8) return fail(MQ_ERR_INVALID, "per-layer bits need parent (8-plane) blobs");
    if (B < 1 || B > 16) return fail(MQ_ERR_INVALID, "stack decode batch %d outside [1, 16]", B);
    StackPlanHost* P = reinterpret_cast<StackPlanHost*>(plan_host);
    mq::StackLayer* T = reinterpret_cast<mq::StackLayer*>(table_host);
    memset(P, 0, sizeof(*P));
    const int nt = B <= 8 ? 1 : 2;
    int cs_max = 1, nstage_max = 1, r_first = 0, nsteps_max = 1, cl_tiles = 0, nrt_max = 1;
    bool zp_any = false, uniform = true;
    size_t partials = 0, stage_max = 0, ll_bytes = 0;
    int n_tickets = 0, n_pair_layers = 0, res_k = 0, res_k_max = 0;
    std::vector<int> res_pub((size_t)n_layers, 0);
    std::vector<int> war((size_t)n_layers, -1);
    // staging holds the most copies any layer stages and the ring the largest
    // stage: every layer's K chunk is sized for both, so any layer fits
    for (int i = 0; i < n_layers; ++i) {
        const int ri = r ? r : layers[i].r;
        if (!valid_r(ri)) return fail(MQ_ERR_INVALID, "layer %d: unsupported bits %d", i, ri);
        // k_stack's staging rule: fp16 decode for r in {4, 8} at nt = 1 (copies at
        // offsets {0, 4} / {0}), else the bf16 zero-point copies
        // (round 1 reserved one more copy for the fp16 path's two-pass staging; dropping it
        // took B = 8 r = 4 2.71 -> 1.80 ms and r = 8 4.83 -> 2.63 ms, neutral at B = 1)
        const bool f16 = mq::stack_f16(ri, nt);
        const int ncopy = f16 ? (ri == 4 ? 2 : 1) : (mq::stack_zp(ri, nt) ? mq::zp_ncopies(ri) : 1);
        nstage_max = std::max(nstage_max, ncopy);
        // k_stack's ZP rule (r = 6: one copy, constants still needed)
        zp_any = zp_any || mq::stack_zp(ri, nt);
        // budget the ring as if for a parent slice (r + 1 planes) even for children,
        // so a child stack gets its parent's decomposition (same summation order)
        const int npl_budget = ri == 8 ? 8 : ri + 1;
        stage_max = std::max(stage_max, (size_t)npl_budget * 512 + 128);
        nsteps_max = std::max(nsteps_max, mq::pad256(std::max(layers[i].K, 1)) / 256);
        if (layers[i].xop == MQ_XOP_ADD_RMSNORM) res_k_max = std::max(res_k_max, layers[i].K);
        nrt_max = std::max(nrt_max, mq::pad16(std::max(layers[i].N, 1)) / 16);
    }
    // CTA-pair reduction slots: at most ceil(n_rt / (sms / 2)) tiles per CTA
    const int cl_max = pair ? 2 * mq::cdiv(nrt_max, std::max(1, sm_count() / 2)) : 0;  // two buffers
    const size_t cl_reserve = cl_max ? (size_t)32 * cl_max + (size_t)cl_max * 32 * nt * 16 : 0;
    // everything but the activation chunk: table, partial slots, zero-point
    // constants, barriers, a 2-deep ring
    // [kept residual B x K bf16][row-group sums B x K/128] (+ a K fp32 copy of the RMSNorm
    // weight when the one-chunk staging still fits beside it: read at staging time without
    // an L2 round trip)
    size_t res_bytes = res_k_max ? (((size_t)B * res_k_max * 2 + 15) & ~(size_t)15) +
                                       (((size_t)B * (res_k_max / 128) * 4 + 15) & ~(size_t)15) + 16
                                 : 0;
    size_t other = res_bytes + sizeof(mq::StackLayer) * (size_t)n_layers + (size_t)mq::kStackWarps * 32 * nt * 16 +
                   (zp_any ? (size_t)2 * nsteps_max * nt * 32 : 0) + cl_reserve + mq::kStackWarps * 128 + (size_t)2 * mq::kStackWarps * stage_max + 256;
    size_t nw_bytes = 0;
    if (res_k_max) {
        const size_t need_xs = (size_t)nstage_max * B * (mq::pad256(res_k_max) + 8) * 2;
        const size_t nw = (size_t)res_k_max * 4 + 16;
        if (other + need_xs + nw <= kSmemFullSm) {
            nw_bytes = nw;
            other += nw;
        }
    }
    // the activation chunk's cap keeps B <= 4 stacks on the measured-best decompositions;
    // B >= 5 would otherwise split K > 2 ways (global split-K tails) -- the ring needs only
    // 2 stages (scripts/sweep_stages.sh), so give staging the rest (B = 8, r = 4: 3.17 ->
    // 2.04 ms/step)
    // Measured on the Llama-3.1-8B stack (MQ_STACK_XS_CAP_KB sweep 40..192 KB per B and r):
    // a smaller cap moves the big-K layers to other K splits; best per batch: 48 KB at
    // B = 1 / 3 and B = 2 r = 2, 64 KB at B = 2 r >= 3 and B = 4 (B = 2 r = 2 1.448 ->
    // 1.335 ms, B = 3 r = 4 1.607 -> 1.494, B = 4 r = 4 1.709 -> 1.581 vs the earlier 80 KB)
    size_t xs_cap = (size_t)192 * 1024;
    if (B == 1 || B == 3 || (B == 2 && r == 2)) xs_cap = (size_t)48 * 1024;
    else if (B <= 4) xs_cap = (size_t)64 * 1024;
    if (const char* e = getenv("MQ_STACK_XS_CAP_KB")) xs_cap = (size_t)atoi(e) * 1024;  // tuning
    if (res_k_max)  // an add + RMSNorm prologue stages its whole row in one chunk
        xs_cap = std::max(xs_cap, (size_t)nstage_max * B * (mq::pad256(res_k_max) + 8) * 2);
    const size_t xs_budget = std::min<size_t>(xs_cap, kSmemFullSm - std::min(other, kSmemFullSm));
    for (int i = 0; i < n_layers; ++i) {
        const mq_stack_layer& in = layers[i];
        const int ri = r ? r : in.r;
        if (!valid_r(ri)) return fail(MQ_ERR_INVALID, "layer %d: unsupported bits %d", i, ri);
        if (nplanes < ri || nplanes > 8 || (nplanes != ri && nplanes < ri + 1))
            return fail(MQ_ERR_INVALID, "cannot slice %d bits out of %d planes", ri, nplanes);
        if (!in.blob || !in.X || !in.Y) return fail(MQ_ERR_INVALID, "layer %d: null pointer", i);
        if (in.N < 1 || in.K < 1 || (in.K & 7) || in.ldx < in.K || in.ldy < (in.yop == MQ_YOP_SILU_PAIRS ? in.N / 2 : in.N) || (in.ldx & 7) ||
            (reinterpret_cast<uintptr_t>(in.X) & 15))
            return fail(MQ_ERR_INVALID, "layer %d: bad shape / alignment", i);
        if (in.xop < MQ_XOP_NONE || in.xop > MQ_XOP_SILU_MUL) return fail(MQ_ERR_INVALID, "layer %d: bad xop", i);
        if (in.yop != MQ_YOP_NONE && in.yop != MQ_YOP_SILU_PAIRS) return fail(MQ_ERR_INVALID, "layer %d: bad yop", i);
        if (in.yop == MQ_YOP_SILU_PAIRS && ((in.N & 15) || in.ldy < in.N / 2))
            return fail(MQ_ERR_INVALID, "layer %d: gated output needs N %% 16 == 0 and ldy >= N / 2", i);
        if (in.xop == MQ_XOP_SILU_MUL && in.ldx < 2 * in.K)
            return fail(MQ_ERR_INVALID, "layer %d: SiLU gating reads [g | u] of 2 K columns", i);
        if (in.xop == MQ_XOP_ADD_RMSNORM) {
            if (!in.norm_w || (in.K & 127) || (reinterpret_cast<uintptr_t>(in.norm_w) & 15))
                return fail(MQ_ERR_INVALID, "layer %d: add-RMSNorm needs a 16-byte aligned norm_w, K %% 128 == 0", i);
            if ((in.res_in || in.res_out) && (in.ldres < in.K || (in.ldres & 7)))
                return fail(MQ_ERR_INVALID, "layer %d: bad residual stride", i);
            if (!in.res_in && (res_k == 0 || res_k != in.K))
                return fail(MQ_ERR_INVALID, "layer %d: no kept residual of width %d before it", i, in.K);
            for (int j = 0; j < i; ++j)
                if (in.res_in && stack_overlap(in.res_in, in.ldres, in.K, layers[j].Y, layers[j].ldy, stack_out_width(layers[j]), B))
                    return fail(MQ_ERR_INVALID, "layer %d: the residual is written inside the stack", i);
            res_k = in.K;
        }
        if (i == 0) r_first = ri;
        uniform = uniform && ri == r_first;
        const bool child = nplanes == ri;
        const int npl = (child || ri == 8) ? ri : ri + 1;
        StackCfg c = choose_stack_config(in.N, in.K, B, nstage_max, sm_count(), xs_budget, pair,
                                         in.xop == MQ_XOP_ADD_RMSNORM);
        // Small layers (K <= 4096, N <= 6144: Llama's qkv and o) as CTA-pair K halves beat one
        // stream-K chunk: the stream-K boundary exchange and the 1-2 tiles per CTA cost more
        // than the DSMEM reduction (Llama stack B = 1: r = 4 1.351 -> 1.320 ms, r = 2 1.215 ->
        // 1.180, r = 3 1.317 -> 1.279; B = 2 r = 4 1.490 -> 1.425).  Larger layers keep the
        // cost model's choice.  MQ_STACK_FORCE_PAIR_K / _N override the limits (tuning).
        const char* fpk = getenv("MQ_STACK_FORCE_PAIR_K");
        const char* fpn = getenv("MQ_STACK_FORCE_PAIR_N");
        const int pair_k = fpk ? atoi(fpk) : 4096, pair_n = fpn ? atoi(fpn) : 6144;
        {
            const int nst = mq::pad256(in.K) / 256;
            // (not at r = 8, B = 1: one chunk balances its 8-plane steps, 1.637 -> 1.618 ms;
            // at B = 2 the pairs still win, 1.748 -> 1.735)
            const int cs = mq::cdiv(nst, 2);
            // only where the half-K chunk fits the staging budget (which accounts for the
            // layer table: the 224 unfused C3 linears at B = 4 otherwise left no weight ring)
            const bool fits = (size_t)nstage_max * B * (cs * 256 + 8) * 2 <= xs_budget;
            if (pair && fits && !(ri == 8 && B == 1) && in.K <= pair_k && in.N <= pair_n && nst >= 2 &&
                in.xop != MQ_XOP_ADD_RMSNORM)
                c = StackCfg{2, cs, std::min(sm_count() / 2, mq::pad16(in.N) / 16)};
        }
        if (in.xop == MQ_XOP_ADD_RMSNORM && c.S != 1)
            return fail(MQ_ERR_INVALID, "layer %d: the fused prologue's row does not fit the staging area", i);
        const mq::Layout L = mq::Layout::make(in.N, in.K, 128, nplanes);
        mq::StackLayer& t = T[i];
        memset(&t, 0, sizeof(t));
        if (war[(size_t)i] == i) t.ext_pub = 1;
        t.blob = in.blob;
        t.step_words = L.step_words;
        t.X = reinterpret_cast<const uint16_t*>(in.X);
        t.Y = reinterpret_cast<uint16_t*>(in.Y);
        t.ldx = in.ldx;
        t.ldy = in.ldy;
        t.N = in.N;
        t.Np = L.Np;
        t.K = in.K;
        t.nsteps = L.nsteps;
        t.n_rt = L.n_rt;
        t.S = c.S;
        t.cs = c.cs;
        t.cpc = c.cpc;
        t.out_scale = in.out_scale;
        t.xop = in.xop;
        t.res_in = reinterpret_cast<const uint16_t*>(in.res_in);
        t.res_out = reinterpret_cast<uint16_t*>(in.res_out);
        t.norm_w = in.norm_w;
        t.ldres = in.ldres;
        t.eps = in.eps;
        t.yop = in.yop;
        t.r = ri;
        t.stage_bytes = npl * 512 + 128;
        t.xll = -1;
        t.yll = -1;
        t.war_wait = -1;
        if (in.xop == MQ_XOP_ADD_RMSNORM && in.res_out)  // over the residual an earlier layer read
            for (int k = 0; k <= i; ++k)
                if (layers[k].xop == MQ_XOP_ADD_RMSNORM && layers[k].res_in &&
                    stack_overlap(layers[k].res_in, layers[k].ldres, layers[k].K, in.res_out, in.ldres, in.K, B)) {
                    war[(size_t)i] = std::max(war[(size_t)i], k);
                    res_pub[(size_t)k] = 1;
                }
        size_t e = 0;
        const int j = stack_x_producer(layers, i, B, &e);
        if (j == -2)
            return fail(MQ_ERR_INVALID, "layer %d reads part of an earlier layer's output in another layout", i);
        if (j >= 0) {
            if (T[j].yll < 0) {  // j's output gets LL words: [B][pad16(N_j) / 2]
                T[j].yll = (long long)(ll_bytes / 8);
                T[j].ldyll = (T[j].yop == MQ_YOP_SILU_PAIRS ? T[j].Np / 2 : T[j].Np) / 2;
                ll_bytes += (size_t)B * T[j].ldyll * 8;
            }
            t.xll = T[j].yll + (long long)(e / 2);
            t.ldxll = T[j].ldyll;
        } else {
            // activations from outside the step: a later layer overwriting them waits
            // until every CTA staged them
            for (int k = i; k < n_layers; ++k)
                if (stack_overlap(in.X, in.ldx, in.K, layers[k].Y, layers[k].ldy, stack_out_width(layers[k]), B)) {
                    t.ext_pub = 1;
                    war[(size_t)k] = std::max(war[(size_t)k], i);
                }
        }
        cs_max = std::max(cs_max, c.cs);
        if (c.S == 1) {  // stream-K: pairs [c fq + min(c, fr), ...), boundary parts through LL words
            const long long P = (long long)L.n_rt * L.nsteps;
            t.flat = 1;
            t.fq = (int)(P / sm_count());
            t.fr = (int)(P % sm_count());
            t.fl_off = (long long)(ll_bytes / 8);
            ll_bytes += (size_t)sm_count() * 32 * nt * 4 * 8;
        }
        if (pair && c.S == 2) {
            cl_tiles = std::max(cl_tiles, mq::cdiv(L.n_rt, c.cpc));
            t.cl_base = n_pair_layers++ & 1;  // buffer index; scaled to slots below
        }
        if (c.S > 1 && !(pair && c.S == 2)) {  // this layer's own partials and tickets
            t.ws_off = (long long)(partials / sizeof(float));
            partials += (size_t)c.S * B * L.Np * sizeof(float);
            t.tk_off = n_tickets;
            n_tickets += L.n_rt;
        }
    }
    for (int i = 0; i < n_layers; ++i) {
        T[i].war_wait = war[(size_t)i];
        if (res_pub[(size_t)i]) T[i].ext_pub = 1;
        T[i].cl_base *= cl_tiles;  // two slot buffers of cl_tiles each
    }
    cl_tiles *= 2;
    mq::StackParams& p = P->p;
    p.n_layers = n_layers;
    p.B = B;
    p.xs_stride = cs_max * 256 + 8;
    p.xcopy_stride = B * p.xs_stride;
    p.cs_off = (int)(((size_t)nstage_max * p.xcopy_stride * 2 + 15) & ~(size_t)15);
    // [2 groups per step][nt * 8 rows] floats; fp16 layers {c / lambda, 1 / lambda} pairs
    const size_t zc_bytes = zp_any ? (size_t)2 * cs_max * nt * 8 * 4 * 2 : 0;
    p.slot_off = (int)((p.cs_off + zc_bytes + 15) & ~(size_t)15);
    const size_t slot_bytes = (size_t)mq::kStackWarps * 32 * nt * 4 * sizeof(float);
    p.table_off = (int)((p.slot_off + slot_bytes + 15) & ~(size_t)15);
    p.res_k = res_k_max;
    p.xops = 0;
    for (int i = 0; i < n_layers; ++i) p.xops |= layers[i].xop != MQ_XOP_NONE || layers[i].yop != MQ_YOP_NONE;
    if (p.xops && (nt != 1 || nplanes != 8))
        return fail(MQ_ERR_INVALID, "fused activation prologues need B <= 8 and parent layers");
    p.res_off = (int)((p.table_off + sizeof(mq::StackLayer) * (size_t)n_layers + 15) & ~(size_t)15);
    p.rpart_off = (int)((p.res_off + (size_t)B * res_k_max * 2 + 15) & ~(size_t)15);
    const int nw_at = (int)((p.rpart_off + (size_t)B * (res_k_max / 128) * 4 + 15) & ~(size_t)15);
    p.nw_off = nw_bytes ? nw_at : 0;
    p.cl_off = (int)((nw_at + (nw_bytes ? (size_t)res_k_max * 4 : 0) + 15) & ~(size_t)15);
    p.cluster = pair ? 1 : 0;
    p.cl_tiles = cl_tiles;
    // [full mbarriers, uses | free mbarriers, free uses] (32 B per tile) + the partial slots
    const size_t cl_bytes = cl_tiles ? (size_t)32 * cl_tiles + (size_t)cl_tiles * 32 * nt * 16 : 0;
    p.xs_bytes = (int)((p.cl_off + cl_bytes + 15) & ~(size_t)15);
    const size_t fixed = (size_t)p.xs_bytes + mq::kStackWarps * 8 * 16;  // full + empty barriers
    const int d = (int)((kSmemFullSm - std::min(fixed, kSmemFullSm)) / (mq::kStackWarps * stage_max));
    if (d < 2) return fail(MQ_ERR_INVALID, "stack: activation staging leaves no room for the weight ring");
    p.stages = std::min(8, d);
    if (const char* e = getenv("MQ_STACK_MAX_STAGES")) p.stages = std::max(2, std::min(p.stages, atoi(e)));  // tuning
    p.stage_stride = (int)stage_max;
    P->smem = fixed + (size_t)mq::kStackWarps * p.stages * stage_max;
    P->r = uniform ? r_first : 0;  // 0: the per-layer dispatch kernel
    P->nplanes = nplanes;
    P->nt = nt;
    P->grid = sm_count();
    size_t od, ol, op;
    P->ll_bytes = ll_bytes;
    P->tk_bytes = (size_t)n_tickets * sizeof(int);
    P->ws_bytes = stack_ws_layout(n_layers, ll_bytes, partials, &od, &ol, &op, P->tk_bytes);
    *workspace_bytes = P->ws_bytes;
    return MQ_OK;
}

int mq_stack_plan(const mq_stack_layer* layers, int n_layers, int B, int r, int nplanes, void* plan_host,
                  void* table_host, size_t* workspace_bytes) {
    const char* env = getenv("MQ_STACK_PAIR");
    bool pair = sm_count() % 2 == 0 && !(env && env[0] == '0');
    // two n-tiles (B > 8) at r >= 3, and r = 8 at B = 8: the pair slots' shared memory costs
    // the staging more than the DSMEM reduction saves (B = 16 r = 4 4.10 -> 2.98 ms, r = 8
    // 21.5 -> 4.5 ms; B = 8 r = 8 2.63 -> 2.38 ms without pairs; r = 2 at B = 16 and every
    // r < 8 at B <= 8 keep them)
    if (((B > 8 && r != 2) || (B == 8 && r == 8)) && r != 0 && !(env && env[0] == '1')) pair = false;
    // per-layer r (r = 0) at B = 1: no pairs either (the 224-linear C3 stack 2.022 -> 1.978
    // ms, a fused ladder mix 1.604 -> 1.595; at B = 2 the pairs win, 2.895 -> 2.143)
    if (r == 0 && B == 1 && !(env && env[0] == '1')) pair = false;
    // r = 8 at B = 1: none (stack 1.617 -> 1.612 ms; the decoder's per-block segments
    // 436 -> 444 tok/s, scripts/full_pair_ab.sh)
    if (r == 8 && B == 1 && !(env && env[0] == '1')) pair = false;
    // the decoder's block segments (fused prologues) at r = 2, B = 1: none (full decode
    // 556 -> 562 tok/s; the bare stack at r = 2 keeps them, 1.180 vs 1.213 ms)
    bool xops = false;
    for (int i = 0; i < n_layers && layers; ++i) xops = xops || layers[i].xop != MQ_XOP_NONE || layers[i].yop != MQ_YOP_NONE;
    if (xops && r == 2 && B == 1 && !(env && env[0] == '1')) pair = false;
    int st = stack_plan_impl(layers, n_layers, B, r, nplanes, plan_host, table_host, workspace_bytes, pair);
    if (st || !pair) return st;
    const StackPlanHost* P = reinterpret_cast<const StackPlanHost*>(plan_host);
    if (mq::stack_pair_capacity(P->nt, P->r, P->nplanes == P->r, P->smem, P->p.xops) >= P->grid &&
        mq::stack_probe(P->nt, P->r, P->nplanes == P->r, P->grid, P->smem, true, P->p.xops) == cudaSuccess)
        return MQ_OK;
    // pairs cannot all be resident (or the driver rejects a cooperative cluster
    // launch): plain cooperative CTAs, global split-K
    st = stack_plan_impl(layers, n_layers, B, r, nplanes, plan_host, table_host, workspace_bytes, false);
    if (st) return st;
    if (mq::stack_probe(P->nt, P->r, P->nplanes == P->r, P->grid, P->smem, false, P->p.xops) != cudaSuccess)
        return fail(MQ_ERR_CUDA, "mq_stack_plan: the persistent kernel cannot be launched cooperatively "
                                 "(%d CTAs, %zu B shared memory)", P->grid, P->smem);
    return MQ_OK;
}

int mq_stack_run(const void* plan_host, const void* table_dev, void* workspace, size_t workspace_bytes,
                 void* stream) {
    if (!plan_host || !table_dev || !workspace) return fail(MQ_ERR_INVALID, "null pointer");
    const StackPlanHost* P = reinterpret_cast<const StackPlanHost*>(plan_host);
    if (workspace_bytes < P->ws_bytes)
        return fail(MQ_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, P->ws_bytes);
    mq::StackParams p = P->p;
    size_t od, ol, op;
    stack_ws_layout(p.n_layers, P->ll_bytes, 0, &od, &ol, &op, P->tk_bytes);
    char* w = reinterpret_cast<char*>(workspace);
    p.layers = reinterpret_cast<const mq::StackLayer*>(table_dev);
    p.tickets = reinterpret_cast<int*>(w);
    p.done = reinterpret_cast<unsigned long long*>(w + od);
    p.launch_ctr = p.done + p.n_layers;
    p.ll = reinterpret_cast<unsigned long long*>(w + ol);
    p.ws = reinterpret_cast<float*>(w + op);
#ifdef MQ_GEMV_TIMING
    static unsigned long long* sbuf = nullptr;
    if (!sbuf) cudaMalloc(&sbuf, sizeof(unsigned long long) * (256 * 148 * 8 + 256 * 16 * 4) + 65536);
    p.dbg_ts = sbuf;
    g_stack_dbg = sbuf;
#endif
    const bool child = P->nplanes == P->r;
    cudaError_t e;
    switch (P->r) {
        case 0: e = mq::launch_stack_mixed(p, P->nt, P->grid, P->smem, (cudaStream_t)stream); break;
        case 2: e = mq::launch_stack_r<2>(p, P->nt, child, P->grid, P->smem, (cudaStream_t)stream); break;
        case 3: e = mq::launch_stack_r<3>(p, P->nt, child, P->grid, P->smem, (cudaStream_t)stream); break;
        case 4: e = mq::launch_stack_r<4>(p, P->nt, child, P->grid, P->smem, (cudaStream_t)stream); break;
        case 6: e = mq::launch_stack_r<6>(p, P->nt, child, P->grid, P->smem, (cudaStream_t)stream); break;
        default: e = mq::launch_stack_r<8>(p, P->nt, child, P->grid, P->smem, (cudaStream_t)stream); break;
    }
    return cuda_status(e, "mq_stack_run");
}

// The step counter: launch_ctr = launches * grid between steps (it also gives
// the LL tag of each step), done[l] the external-staging counters.  set = 1
// writes `*launches` to all of them and clears the LL words, so a re-based
// counter can never meet a stale tag (tests seed it near 2^32 to show the
// 64-bit counters do not wrap); set = 0 reads it back.  Synchronous.
int mq_stack_epoch(const void* plan_host, void* workspace, size_t workspace_bytes, unsigned long long* launches,
                   int set, void* stream) {
    if (!plan_host || !workspace || !launches) return fail(MQ_ERR_INVALID, "null pointer");
    const StackPlanHost* P = reinterpret_cast<const StackPlanHost*>(plan_host);
    if (workspace_bytes < P->ws_bytes)
        return fail(MQ_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, P->ws_bytes);
    size_t od, ol, op;
    stack_ws_layout(P->p.n_layers, P->ll_bytes, 0, &od, &ol, &op, P->tk_bytes);
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(workspace) + od);
    const int n = P->p.n_layers + 1;
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<unsigned long long> h((size_t)n);
    const unsigned long long grid = (unsigned long long)P->grid;
    cudaError_t e;
    if (set) {
        for (auto& v : h) v = *launches * grid;
        e = cudaMemcpyAsync(ctr, h.data(), sizeof(unsigned long long) * n, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess && P->ll_bytes)
            e = cudaMemsetAsync(reinterpret_cast<char*>(workspace) + ol, 0, P->ll_bytes, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        return cuda_status(e, "mq_stack_epoch");
    }
    e = cudaMemcpyAsync(h.data(), ctr, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "mq_stack_epoch");
    const unsigned long long lc = h[(size_t)n - 1];
    for (int i = 0; i < n; ++i)
        if (h[i] > lc || h[i] % grid)
            return fail(MQ_ERR_INVALID, "stack counters inconsistent (layer %d: %llu vs %llu)", i, h[i], lc);
    *launches = lc / grid;
    return MQ_OK;
}

static int sync_and_check(cudaError_t launch, int* err_dev, cudaStream_t s, const char* where,
                          const char* range_msg) {
    if (launch != cudaSuccess) return cuda_status(launch, where);
    int h = 0;
    cudaError_t e = cudaMemcpyAsync(&h, err_dev, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, where);
    if (h) return fail(MQ_ERR_CODE_RANGE, "%s", range_msg);
    return MQ_OK;
}

int mq_slice_elementwise(const uint8_t* q, long long n, int c, int r, int on_master, uint8_t* out,
                         int* err_dev, void* stream) {
    if (c < 2 || c > 8) return fail(MQ_ERR_INVALID, "master bit-width must lie in [2, 8]");
    if (r > c) return fail(MQ_ERR_INVALID, "cannot slice %d bits out of %d", r, c);
    if (r < 2) return fail(MQ_ERR_INVALID, "target bit-width must be >= 2");
    if (n < 0 || (n > 0 && (!q || !out || !err_dev))) return fail(MQ_ERR_INVALID, "null pointer");
    if (n == 0) return MQ_OK;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(err_dev, 0, sizeof(int), s);
    if (e != cudaSuccess) return cuda_status(e, "mq_slice_elementwise");
    static char msg[64];
    snprintf(msg, sizeof(msg), "code out of range for bit-width %d", c);
    return sync_and_check(mq::launch_slice_elementwise(q, n, c, r, on_master, out, err_dev, s),
                          err_dev, s, "mq_slice_elementwise", msg);
}

int mq_dequant_f64(const uint8_t* codes, int N, int K, const float* scales, int ng, int G, int c,
                   int r, double* out, int* err_dev, void* stream) {
    if (c < 2 || c > 8 || r < 2 || r > c) return fail(MQ_ERR_INVALID, "bad bit-widths c=%d r=%d", c, r);
    if (N < 1 || K < 1 || G < 1 || ng < mq::cdiv(K, G)) return fail(MQ_ERR_INVALID, "bad shape");
    if (!codes || !scales || !out || !err_dev) return fail(MQ_ERR_INVALID, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(err_dev, 0, sizeof(int), s);
    if (e != cudaSuccess) return cuda_status(e, "mq_dequant_f64");
    static char msg[64];
    snprintf(msg, sizeof(msg), "code out of range for bit-width %d", r);
    return sync_and_check(mq::launch_dequant_f64(codes, N, K, scales, ng, G, c, r, out, err_dev, s),
                          err_dev, s, "mq_dequant_f64", msg);
}

int mq_dequant_value_f64(const uint8_t* q, const double* scale, long long n, int c, int r,
                         double* out, int* err_dev, void* stream) {
    if (c < 2 || c > 8 || r < 2 || r > c) return fail(MQ_ERR_INVALID, "bad bit-widths c=%d r=%d", c, r);
    if (n < 0 || (n > 0 && (!q || !scale || !out || !err_dev))) return fail(MQ_ERR_INVALID, "null pointer");
    if (n == 0) return MQ_OK;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(err_dev, 0, sizeof(int), s);
    if (e != cudaSuccess) return cuda_status(e, "mq_dequant_value_f64");
    static char msg[64];
    snprintf(msg, sizeof(msg), "code out of range for bit-width %d", r);
    return sync_and_check(mq::launch_dequant_value_f64(q, scale, n, c, r, out, err_dev, s), err_dev,
                          s, "mq_dequant_value_f64", msg);
}

int mq_matmul_ref(const float* X, int B, int K, const float* W, int N, float* Y, void* stream) {
    if (!X || !W || !Y) return fail(MQ_ERR_INVALID, "null pointer");
    if (B < 1 || K < 1 || N < 1) return fail(MQ_ERR_INVALID, "bad shape");
    return cuda_status(mq::launch_matmul_ref(X, B, K, W, N, Y, (cudaStream_t)stream), "mq_matmul_ref");
}

int mq_pack_ref_layout(const uint8_t* codes, int N, int K, int bits, uint64_t* base, uint32_t* b2,
                       uint32_t* b3, int* err_dev, void* stream) {
    if (bits < 2 || bits > 4) return fail(MQ_ERR_INVALID, "unsupported bits");
    if (!codes || !base || !err_dev || (bits >= 3 && !b2) || (bits == 4 && !b3))
        return fail(MQ_ERR_INVALID, "null pointer");
    if (N < 1 || K < 1) return fail(MQ_ERR_INVALID, "bad shape");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(err_dev, 0, sizeof(int), s);
    if (e != cudaSuccess) return cuda_status(e, "mq_pack_ref_layout");
    static char msg[64];
    snprintf(msg, sizeof(msg), "code overflow for %d bits", bits);
    return sync_and_check(
        mq::launch_pack_ref_layout(codes, N, K, bits, reinterpret_cast<unsigned long long*>(base),
                                   bits >= 3 ? b2 : nullptr, bits == 4 ? b3 : nullptr, err_dev, s),
        err_dev, s, "mq_pack_ref_layout", msg);
}

int mq_unpack_ref_layout(const uint64_t* base, const uint32_t* b2, const uint32_t* b3, int N, int K,
                         uint8_t* codes, void* stream) {
    if (!base || !codes) return fail(MQ_ERR_INVALID, "null pointer");
    if (N < 1 || K < 1) return fail(MQ_ERR_INVALID, "bad shape");
    return cuda_status(mq::launch_unpack_ref_layout(reinterpret_cast<const unsigned long long*>(base),
                                                    b2, b3, N, K, codes, (cudaStream_t)stream),
                       "mq_unpack_ref_layout");
}

// ---- MatGPTQ quantiser searches ------------------------------------------
static int quant_targets(const int* targets, const double* lams, int T, mq::QuantTargets* tg) {
    if (!targets || !lams || T < 1 || T > 7) return fail(MQ_ERR_INVALID, "bad bit-width set");
    tg->T = T;
    for (int t = 0; t < T; ++t) {
        if (targets[t] < 2 || targets[t] > 8 || (t && targets[t] <= targets[t - 1]))
            return fail(MQ_ERR_INVALID, "bit-widths must be distinct, sorted and in [2, 8]");
        if (!(lams[t] > 0.0) || lams[t] > 1.7976931348623157e308)
            return fail(MQ_ERR_INVALID, "importance weights must be positive and finite");
        tg->r[t] = targets[t];
        tg->lam[t] = lams[t];
    }
    tg->c = targets[T - 1];
    return MQ_OK;
}

int mq_select_codes(const double* W, long long ldw, int d_row, int d_col, const float* scales, int ngs, int G,
                    const int* targets, const double* lams, int T, uint8_t* codes, long long ldc, void* stream) {
    mq::QuantTargets tg;
    if (int st = quant_targets(targets, lams, T, &tg)) return st;
    if (!W || !scales || !codes) return fail(MQ_ERR_INVALID, "null pointer");
    if (d_row < 0 || d_col < 0 || G < 1 || ldw < d_col || ldc < d_col || ngs < (d_col + G - 1) / G)
        return fail(MQ_ERR_INVALID, "bad shape");
    if ((long long)d_row * d_col == 0) return MQ_OK;
    return cuda_status(mq::launch_select_codes(W, ldw, d_row, d_col, scales, ngs, G, tg, codes, ldc,
                                               (cudaStream_t)stream),
                       "mq_select_codes");
}

int mq_fit_grid(const double* W, long long ldw, int d_row, int d_col, int G, const int* targets,
                const double* lams, int T, const double* alphas, int steps, float* scales, void* stream) {
    mq::QuantTargets tg;
    if (int st = quant_targets(targets, lams, T, &tg)) return st;
    if (!W || !alphas || !scales) return fail(MQ_ERR_INVALID, "null pointer");
    if (d_row < 1 || d_col < 1) return fail(MQ_ERR_INVALID, "weights must be a non-empty matrix");
    if (steps < 1) return fail(MQ_ERR_INVALID, "steps must be >= 1");
    if (G < 1 || G > 4096 || ldw < d_col) return fail(MQ_ERR_INVALID, "bad shape");
    const int ngs = (d_col + G - 1) / G;
    return cuda_status(mq::launch_fit_grid(W, ldw, d_row, d_col, G, tg, alphas, steps, scales, ngs,
                                           (cudaStream_t)stream),
                       "mq_fit_grid");
}

int mq_rtn_f64(const double* w, const double* scale, long long n, int c, long long* codes, int* err_dev,
               void* stream) {
    if (c < 2 || c > 8) return fail(MQ_ERR_INVALID, "bit-width must lie in [2, 8]");
    if (n < 0 || (n > 0 && (!w || !scale || !codes || !err_dev))) return fail(MQ_ERR_INVALID, "null pointer");
    if (n == 0) return MQ_OK;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(err_dev, 0, sizeof(int), s);
    if (e != cudaSuccess) return cuda_status(e, "mq_rtn_f64");
    return sync_and_check(mq::launch_rtn(w, scale, n, c, 1, nullptr, codes, err_dev, s), err_dev, s, "mq_rtn_f64",
                          "non-finite weight");
}

int mq_round_half_away_f64(const double* x, long long n, double* out, void* stream) {
    if (n < 0 || (n > 0 && (!x || !out))) return fail(MQ_ERR_INVALID, "null pointer");
    if (n == 0) return MQ_OK;
    return cuda_status(mq::launch_rtn(x, nullptr, n, 2, 0, out, nullptr, nullptr, (cudaStream_t)stream),
                       "mq_round_half_away_f64");
}

int mq_gptq_block(double* Wc, long long ldw, int d_row, int d_col, int lo, int hi, const float* scales, int ngs,
                  int G, const double* chol, long long ldch, const int* targets, const double* lams, int T,
                  uint8_t* codes, long long ldc, double* comp, long long ldcomp, double* err, long long lde,
                  void* stream) {
    mq::QuantTargets tg;
    if (int st = quant_targets(targets, lams, T, &tg)) return st;
    if (!Wc || !scales || !chol || !codes || !comp || !err) return fail(MQ_ERR_INVALID, "null pointer");
    if (d_row < 1 || lo < 0 || hi <= lo || hi > d_col || G < 1 || ldw < d_col || ldch < d_col ||
        ldc < d_col || ldcomp < d_col || lde < hi - lo || ngs < (d_col + G - 1) / G)
        return fail(MQ_ERR_INVALID, "bad shape");
    return cuda_status(mq::launch_gptq_block(Wc, ldw, d_row, lo, hi, scales, ngs, G, chol, ldch, tg, codes, ldc,
                                             comp, ldcomp, err, lde, (cudaStream_t)stream),
                       "mq_gptq_block");
}

// ---- full-model harness glue (llama.py) ------------------------------------
int mq_add_rmsnorm(void* x, const void* delta, const float* w, void* y, int B, int h, float eps, void* stream) {
    if (!x || !w || !y) return fail(MQ_ERR_INVALID, "null pointer");
    if (B < 1 || h < 1) return fail(MQ_ERR_INVALID, "bad shape");
    return cuda_status(mq::launch_add_rmsnorm(x, delta, w, y, B, h, eps, (cudaStream_t)stream), "mq_add_rmsnorm");
}

int mq_rope_kv(const void* qkv, const void* cosv, const void* sinv, void* q, void* kcache, void* vcache, int B,
               int n_heads, int n_kv_heads, int head_dim, int T, int pos, void* stream) {
    return mq_qknorm_rope_kv(qkv, cosv, sinv, q, kcache, vcache, B, n_heads, n_kv_heads, head_dim, T, pos, nullptr,
                             nullptr, 0.0f, stream);
}

int mq_qknorm_rope_kv(const void* qkv, const void* cosv, const void* sinv, void* q, void* kcache, void* vcache,
                      int B, int n_heads, int n_kv_heads, int head_dim, int T, int pos, const float* q_norm,
                      const float* k_norm, float eps, void* stream) {
    if (!qkv || !cosv || !sinv || !q || !kcache || !vcache) return fail(MQ_ERR_INVALID, "null pointer");
    if (B < 1 || n_heads < 1 || n_kv_heads < 1 || head_dim % 64 || head_dim > 256 || pos < 0 || pos >= T)
        return fail(MQ_ERR_INVALID, "bad shape");
    if ((q_norm == nullptr) != (k_norm == nullptr)) return fail(MQ_ERR_INVALID, "q_norm and k_norm go together");
    return cuda_status(mq::launch_rope_kv(qkv, cosv, sinv, q, kcache, vcache, B, n_heads, n_kv_heads, head_dim, T,
                                          pos, q_norm, k_norm, eps, (cudaStream_t)stream),
                       "mq_qknorm_rope_kv");
}

int mq_attn_decode(const void* qkv, const void* cosv, const void* sinv, const float* q_norm, const float* k_norm,
                   float eps, void* kcache, void* vcache, const int* kv_of_q, void* att, int B, int n_heads,
                   int n_kv_heads, int head_dim, int T, int pos, void* stream) {
    if (!qkv || !cosv || !sinv || !kcache || !vcache || !kv_of_q || !att) return fail(MQ_ERR_INVALID, "null pointer");
    if (B < 1 || n_heads < 1 || n_kv_heads < 1 || (head_dim != 64 && head_dim != 128) || pos < 0 || pos >= T ||
        pos >= 50 * 1024)
        return fail(MQ_ERR_INVALID, "bad shape (head_dim 64 / 128, 0 <= pos < min(T, 51200))");
    if ((q_norm == nullptr) != (k_norm == nullptr)) return fail(MQ_ERR_INVALID, "q_norm and k_norm go together");
    return cuda_status(mq::launch_attn_decode(qkv, cosv, sinv, q_norm, k_norm, eps, kcache, vcache, kv_of_q, att, B,
                                              n_heads, n_kv_heads, head_dim, T, pos, (cudaStream_t)stream),
                       "mq_attn_decode");
}

int mq_silu_mul(const void* gu, void* y, int B, int inter, void* stream) {
    if (!gu || !y) return fail(MQ_ERR_INVALID, "null pointer");
    if (B < 1 || inter < 1) return fail(MQ_ERR_INVALID, "bad shape");
    return cuda_status(mq::launch_silu_mul(gu, y, B, inter, (cudaStream_t)stream), "mq_silu_mul");
}

}  // extern "C"
