// matq_gemm.cu -- K4 launcher: TMA tensor map for the activations, tile
// grid, template dispatch over (r, child, token tile).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "matq_gemm.cuh"
#include "matq_internal.h"

namespace mq {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

template <int R, bool CHILD, int BN>
cudaError_t launch_bn(const CUtensorMap& map, const GemmParams& p, int grid, cudaStream_t stream,
                      bool pdl) {
    auto kern = k_gemm<R, CHILD, BN>;
    constexpr int smem = (int)GemmSmem<BN, PlaneCount<R, CHILD>::value>::kBytes;
    // once per instantiation; a function-local static is initialised thread-safely
    static const cudaError_t attr_err =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (attr_err != cudaSuccess) return attr_err;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    if (pdl) {
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    return cudaLaunchKernelEx(&cfg, kern, map, p);
}

template <int R, bool CHILD>
cudaError_t launch_rc(int bn, const CUtensorMap& map, const GemmParams& p, int grid,
                      cudaStream_t stream, bool pdl) {
    if (bn == 64) return launch_bn<R, CHILD, 64>(map, p, grid, stream, pdl);
    if (bn == 128) return launch_bn<R, CHILD, 128>(map, p, grid, stream, pdl);
    if constexpr (gemm_bn512_ok(R)) {
        if (bn == 512) return launch_bn<R, CHILD, 512>(map, p, grid, stream, pdl);
    }
    return launch_bn<R, CHILD, 256>(map, p, grid, stream, pdl);
}

}  // namespace

#ifdef MQ_GEMV_TIMING
unsigned long long* gemm_dbg_buffer() {
    static unsigned long long* buf = nullptr;
    if (!buf && cudaMalloc(&buf, sizeof(unsigned long long) * 64 * 160 * 6) == cudaSuccess)
        cudaMemset(buf, 0, sizeof(unsigned long long) * 64 * 160 * 6);
    return buf;
}
#endif

namespace {
// one token-tile width: the split-K / split-tail plan minimising the busiest CTA's steps
GemmConfig plan_gemm(int N, int K, int B, int sms, int bn, double* cost_out) {
    GemmConfig c{};
    c.bn = bn;
    const int n_bt = cdiv(B, c.bn);
    c.n_tiles = cdiv(N, kGemmBM) * n_bt;
    const int nsteps = pad256(K) / 256;
    // K splits only when the tiles leave SMs idle: minimise the busiest CTA's
    // steps (+ ~4 steps of partial write / in-order reduction per split tile).
    double best = 1e30;
    for (int S = 1; S <= std::min(8, nsteps); ++S) {
        const int cs = cdiv(nsteps, S);
        if (cdiv(nsteps, cs) != S) continue;
        const int units = c.n_tiles * S;
        // a split tile costs its partial round trip: ~1.5 steps when every unit is
        // resident (the S splits reduce 1/S of the columns each), ~4 when the last
        // split to arrive reduces the whole tile
        const double fix = S == 1 ? 0.0 : (units <= sms ? 1.5 : 4.0);
        const double cost = (double)cdiv(units, sms) * (cs + fix);
        if (cost < best - 1e-9) {
            best = cost;
            c.S = S;
            c.cs = cs;
        }
    }
    c.t1 = 0;
    // whole waves + a split tail: when the tiles overflow the grid by R < sms, the first
    // floor(n_tiles / sms) waves run whole tiles and the R leftover tiles are split S2
    // ways over the last wave (every split resident: the coop reduction), instead of a
    // nearly empty extra wave of whole tiles (Qwen3-14B o / down at B = 1024: 160 tiles)
    const int waves = c.n_tiles / sms, rem = c.n_tiles - waves * sms;
    if (waves >= 1 && rem > 0) {
        for (int S2 = std::min(8, nsteps); S2 >= 2; --S2) {
            const int cs2 = cdiv(nsteps, S2);
            if (cdiv(nsteps, cs2) != S2 || rem * S2 > sms) continue;
            const double cost = (double)waves * nsteps + cs2 + 1.5;
            if (cost < best - 1e-9) {
                best = cost;
                c.t1 = waves * sms;
                c.S = S2;
                c.cs = cs2;
            }
            break;  // the largest admissible split is the cheapest tail
        }
    }
    const int units = c.t1 + (c.n_tiles - c.t1) * c.S;
    c.grid = std::min(units, sms);
    *cost_out = best;
    return c;
}
}  // namespace

GemmConfig choose_gemm_config(int N, int K, int B, int sms, int r) {
    double cost = 0.0;
    const int bn = B <= 64 ? 64 : (B <= 128 ? 128 : 256);
    GemmConfig c = plan_gemm(N, K, B, sms, bn, &cost);
    // past 256 tokens a 512-token tile decodes each weight tile once for two N = 256
    // MMAs (two operand stages of 80 KB; at r = 8 one raw stage beside them).
    // Its steps are MMA-bound at twice the 256-token step, and 2 operand stages plus a
    // single TMEM accumulator cost ~10% more (measured: 2.2 x); it wins where the
    // halved tile count fills the SMs better (Qwen3-14B o / down at B = 384-512)
    // MQ_GEMM_BN512: 0 = never, 2 = always past 256 tokens (tests: several 512-token
    // units per CTA through the single TMEM accumulator), else the cost model
    static const int bn512 = [] {
        const char* e = getenv("MQ_GEMM_BN512");
        return e && (e[0] == '0' || e[0] == '2') ? e[0] - '0' : 1;
    }();
    if (B > 256 && bn512 && gemm_bn512_ok(r)) {
        double cost512 = 0.0;
        const GemmConfig c512 = plan_gemm(N, K, B, sms, 512, &cost512);
        if (bn512 == 2 || 2.2 * cost512 < cost) c = c512;
    }
    return c;
}

size_t gemm_ws_bytes(const GemmConfig& c) {
    if (c.S <= 1) return 0;
    return kGemmTicketBytes + (size_t)(c.n_tiles - c.t1) * c.S * c.bn * kGemmBM * sizeof(float);
}

cudaError_t launch_gemm(const uint32_t* blob, const Layout& L, const void* X, int ldx, void* Y,
                        int ldy, int B, int r, bool child, float out_scale, bool y_f32,
                        const GemmConfig& c, void* ws, cudaStream_t stream, bool pdl,
                        const char** why) {
    auto enc = encode_fn();
    if (enc == nullptr) {
        *why = "cuTensorMapEncodeTiled unavailable";
        return cudaErrorNotSupported;
    }
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)L.K, (cuuint64_t)B};
    const cuuint64_t strides[1] = {(cuuint64_t)ldx * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kGemmBK, (cuuint32_t)std::min(c.bn, 256)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(X), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        *why = "cuTensorMapEncodeTiled rejected the activation tensor";
        return cudaErrorInvalidValue;
    }
    GemmParams p{};
    p.blob = blob;
    p.step_words = L.step_words;
    p.skip_words = 16 * L.spg - 32;
    p.Y = Y;
    p.ldy = ldy;
    p.B = B;
    p.N = L.N;
    p.K = L.K;
    p.nsteps = L.nsteps;
    p.n_rt = L.n_rt;
    p.n_bt = cdiv(B, c.bn);
    p.n_tiles = c.n_tiles;
    p.S = c.S;
    p.cs = c.cs;
    p.t1 = c.t1;
    if (c.S > 1) {
        p.tickets = reinterpret_cast<int*>(ws);
        p.ws = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + kGemmTicketBytes);
    }
    p.out_scale = out_scale;
    p.y_f32 = y_f32 ? 1 : 0;
    p.coop = (c.S > 1 && (c.n_tiles - c.t1) * c.S <= c.grid) ? 1 : 0;
#ifdef MQ_GEMV_TIMING
    static int dbg_ctr = 0;
    p.dbg_slot = dbg_ctr++ % 64;
    p.dbg_ts = gemm_dbg_buffer();
#endif
    const bool ch = child && r < 8;
    const int bn = c.bn, grid = c.grid;
    switch (r) {
        case 2: return ch ? launch_rc<2, true>(bn, map, p, grid, stream, pdl)
                          : launch_rc<2, false>(bn, map, p, grid, stream, pdl);
        case 3: return ch ? launch_rc<3, true>(bn, map, p, grid, stream, pdl)
                          : launch_rc<3, false>(bn, map, p, grid, stream, pdl);
        case 4: return ch ? launch_rc<4, true>(bn, map, p, grid, stream, pdl)
                          : launch_rc<4, false>(bn, map, p, grid, stream, pdl);
        case 6: return ch ? launch_rc<6, true>(bn, map, p, grid, stream, pdl)
                          : launch_rc<6, false>(bn, map, p, grid, stream, pdl);
        case 8: return launch_rc<8, false>(bn, map, p, grid, stream, pdl);
    }
    *why = "unsupported bit-width";
    return cudaErrorInvalidValue;
}

}  // namespace mq
