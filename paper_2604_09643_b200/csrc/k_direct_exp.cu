// k_direct_exp.cu — direct kernels K1/K2 instantiated for the exp family of the designated kernel (R23).
#include "k_direct_impl.cuh"

PA_DIRECT_FAMILY(exp, KF_EXP)
