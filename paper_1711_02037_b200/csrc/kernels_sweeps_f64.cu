// fp64 instantiation of the persistent sweep kernel (kernels_sweeps.cuh).
#define RNMF_SWEEPS_T double
#include "kernels_sweeps.cuh"
