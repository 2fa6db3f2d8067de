#define MQ_R 3
#include "matq_gemv_inst.cuh"
