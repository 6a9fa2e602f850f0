// k_direct_gauss.cu — direct kernels K1/K2 instantiated for the gauss family of the designated kernel (R23).
#include "k_direct_impl.cuh"

PA_DIRECT_FAMILY(gauss, KF_GAUSS)
