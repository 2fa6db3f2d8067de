#define MQ_R 8
#include "matq_gemv_inst.cuh"
