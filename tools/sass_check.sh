#!/bin/bash
# compile gls_kernels.cu to a cubin and list per-line SASS / local-memory counts of the engine-0 kernel
# usage: tools/sass_check.sh [extra nvcc flags]
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -cubin "$@" \
  -o /tmp/gls_k.cubin paper_2304_13398_b200/csrc/gls_kernels.cu -Xptxas -v 2>&1 | grep -A2 "sim_kernelILi0ELb1" | tail -2
nvdisasm -g -c /tmp/gls_k.cubin > /tmp/gls_k.sass
python tools/sass_lines.py /tmp/gls_k.sass sim_kernelILi0ELb1 gls_lanes
