// matq_stack.cu -- K3S instantiations and cooperative launcher.
#include <cstdio>
#include <cstdlib>

#include "matq_stack.cuh"

namespace mq {

namespace {
template <int NT, int R, bool CHILD>
cudaError_t set_smem(size_t smem) {
    static int smem_set = 0;
    if ((int)smem > smem_set) {
        cudaError_t e = cudaFuncSetAttribute(k_stack<NT, R, CHILD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        smem_set = (int)smem;
    }
    return cudaSuccess;
}

template <int NT, int R, bool CHILD>
cudaError_t launch_one_stack(const StackParams& p, int grid, size_t smem, cudaStream_t stream) {
    auto kern = k_stack<NT, R, CHILD>;
    cudaError_t e = set_smem<NT, R, CHILD>(smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kStackThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the layer barriers spin
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    // CTA pairs launch as clusters without the cooperative attribute (the pair is
    // not expressible in a cooperative launch under every tool, e.g. ncu's kernel
    // replay); co-residency of every pair was checked by the plan
    // (stack_pair_capacity >= grid) and the grid never exceeds one CTA per SM
    if (p.cluster) {
        cfg.attrs = attr + 1;
        cfg.numAttrs = 1;
    } else {
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    e = cudaLaunchKernelEx(&cfg, kern, p);
    if (getenv("MQ_STACK_LAUNCH_DEBUG"))
        fprintf(stderr, "k_stack launch cluster=%d grid=%d smem=%zu -> %s\n", p.cluster, grid, smem,
                cudaGetErrorString(e));
    return e;
}

template <int NT, int R, bool CHILD>
int pair_capacity(size_t smem) {
    if (set_smem<NT, R, CHILD>(smem) != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(kStackThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_stack<NT, R, CHILD>, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return 2 * n;
}
}  // namespace

template <int R>
cudaError_t launch_stack_r(const StackParams& p, int nt, bool child, int grid, size_t smem,
                           cudaStream_t stream) {
    constexpr bool kChildOk = R < 8;
    if (child && kChildOk) {
        if (nt == 1) return launch_one_stack<1, R, kChildOk>(p, grid, smem, stream);
        return launch_one_stack<2, R, kChildOk>(p, grid, smem, stream);
    }
    if (nt == 1) return launch_one_stack<1, R, false>(p, grid, smem, stream);
    return launch_one_stack<2, R, false>(p, grid, smem, stream);
}

cudaError_t launch_stack_mixed(const StackParams& p, int nt, int grid, size_t smem, cudaStream_t stream) {
    if (nt == 1) return launch_one_stack<1, 0, false>(p, grid, smem, stream);
    return launch_one_stack<2, 0, false>(p, grid, smem, stream);
}

int stack_pair_capacity(int nt, int r, bool child, size_t smem) {
    const bool c = child && r < 8;
#define MQ_CAP(R)                                                                   \
    if (r == R) {                                                                   \
        if (nt == 1) return c ? pair_capacity<1, R, (R < 8)>(smem) : pair_capacity<1, R, false>(smem); \
        return c ? pair_capacity<2, R, (R < 8)>(smem) : pair_capacity<2, R, false>(smem);             \
    }
    MQ_CAP(2) MQ_CAP(3) MQ_CAP(4) MQ_CAP(6) MQ_CAP(8)
#undef MQ_CAP
    return nt == 1 ? pair_capacity<1, 0, false>(smem) : pair_capacity<2, 0, false>(smem);
}

template cudaError_t launch_stack_r<2>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<3>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<4>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<6>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<8>(const StackParams&, int, bool, int, size_t, cudaStream_t);

}  // namespace mq
