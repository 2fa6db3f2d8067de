// matq_stack.cu -- K3S instantiations and cooperative launcher.
#include "matq_stack.cuh"

namespace mq {

namespace {
template <int NT, int R, bool CHILD>
cudaError_t launch_one_stack(const StackParams& p, int grid, size_t smem, cudaStream_t stream) {
    auto kern = k_stack<NT, R, CHILD>;
    static int smem_set = 0;
    if ((int)smem > smem_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        smem_set = (int)smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kStackThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the layer barriers spin
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
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

template cudaError_t launch_stack_r<2>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<3>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<4>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<6>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<8>(const StackParams&, int, bool, int, size_t, cudaStream_t);

}  // namespace mq
