// fp32 instantiation of the persistent sweep kernel (kernels_sweeps.cuh); one translation unit per
// precision so the two compile in parallel.
#define RNMF_SWEEPS_T float
#define RNMF_SWEEPS_COMMON
#include "kernels_sweeps.cuh"
