#define MQ_R 6
#include "matq_gemv_inst.cuh"
