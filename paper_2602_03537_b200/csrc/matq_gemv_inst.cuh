#include <mutex>
// Per-bit-width instantiation of the K3 launcher (included by matq_gemv_r*.cu
// with MQ_R defined, so the five ladder widths compile in parallel).
#include "matq_gemv.cuh"

namespace mq {

template <typename K>
static cudaError_t launch_one(K kernel, const GemvParams& p, dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, bool pdl, int& smem_set) {
    {
        // the limit only grows; serialised so a smaller request cannot lower it under a
        // concurrent larger one (host threads may launch concurrently)
        static std::mutex mu;
        std::lock_guard<std::mutex> lk(mu);
        if ((int)smem > smem_set) {
            cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
            smem_set = (int)smem;
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (p.pair) {  // CTA pairs: chunk 1 of a tile ships its partial to chunk 0 through DSMEM
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 2;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kernel, p);
}

template <>
cudaError_t launch_gemv_r<MQ_R>(const GemvParams& p, int nt, bool child, int gs, dim3 grid,
                                dim3 block, size_t smem, cudaStream_t stream, bool pdl) {
    constexpr int R = MQ_R;
    constexpr bool kChildOk = R < 8;  // at r = 8 a child is the parent
    static int smem_set[3][2][2] = {};
    const int ni = nt == 1 ? 0 : (nt == 2 ? 1 : 2);
    const int ci = (child && kChildOk) ? 1 : 0;
    const int gi = gs == 128 ? 0 : 1;
    int& ss = smem_set[ni][ci][gi];
#define MQ_L(NT_, CH_, GS_) \
    return launch_one(k_gemv<R, NT_, (CH_ && kChildOk), GS_>, p, grid, block, smem, stream, pdl, ss)
#define MQ_GS(NT_, CH_)          \
    if (gi == 0) MQ_L(NT_, CH_, 128); \
    MQ_L(NT_, CH_, 0)
#define MQ_CH(NT_)                                  \
    if (ci == 1) { MQ_GS(NT_, true); }              \
    MQ_GS(NT_, false)
    if (ni == 0) { MQ_CH(1); }
    if (ni == 1) { MQ_CH(2); }
    MQ_CH(4);
#undef MQ_CH
#undef MQ_GS
#undef MQ_L
}

}  // namespace mq
