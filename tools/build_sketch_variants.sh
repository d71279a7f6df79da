#!/bin/bash
# Builds tools/sketch_acc in several experiment variants (development aid): which resource bounds
# the 3xTF32 X-streaming kernels.  Usage: tools/build_sketch_variants.sh; run tools/sv/* on the GPU.
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/sv
C=paper_1711_02037_b200/csrc
build() { # name flags...
  local name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I $C "$@" \
    tools/sketch_acc.cu $C/kernels_tc.cu $C/kernels_xw.cu $C/kernels_xgemm.cu -o tools/sv/$name &
}
build base
build smem188 -DRNMF_TC_SMEM_KB=188
build lo2 -DRNMF_TC_LO_SLOTS=2
build nosplit -DRNMF_TC_DBG_NOSPLIT
build nolomma -DRNMF_TC_DBG_NOLOMMA
build noslo -DRNMF_TC_DBG_NOSLO
build nosplit_nolomma -DRNMF_TC_DBG_NOSPLIT -DRNMF_TC_DBG_NOLOMMA
build hi_only -DRNMF_TC_DBG_NOSPLIT -DRNMF_TC_DBG_NOLOMMA -DRNMF_TC_DBG_NOSLO
wait
ls -la tools/sv
