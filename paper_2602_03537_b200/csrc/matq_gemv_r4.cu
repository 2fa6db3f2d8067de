#define MQ_R 4
#include "matq_gemv_inst.cuh"
