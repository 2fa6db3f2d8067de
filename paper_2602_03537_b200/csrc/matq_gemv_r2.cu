#define MQ_R 2
#include "matq_gemv_inst.cuh"
