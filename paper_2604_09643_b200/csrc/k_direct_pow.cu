// k_direct_pow.cu — direct kernels K1/K2 instantiated for the pow family of the designated kernel (R23).
#include "k_direct_impl.cuh"

PA_DIRECT_FAMILY(pow, KF_POW)
