#!/bin/bash
# One `ncu --set full` capture per non-GEMM kernel family at a representative size
# (tools/ncu_kernels.py: a warm-up call, then the profiled call inside the NVTX range "prof").
# Run under gpurun; reports land in gpurun_out/ncu_<name>.ncu-rep.
set -u
mkdir -p gpurun_out
run() {  # name regex skip what  (skip: launches of the kernel inside the range to pass over)
  python tools/ncu_kernels.py "$4" > /dev/null 2>&1 || { echo "$1 plain run failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
    -k "regex:$2" --launch-skip "$3" --launch-count 1 \
    -o "gpurun_out/ncu_$1" -f python tools/ncu_kernels.py "$4" > "gpurun_out/ncu_$1.log" 2>&1
  echo "$1 exit $?"
}
run geo 'geo_kernel' 0 geo
run maxvol 'maxvol_kernel' 0 maxvol
run tsqr 'tsqr_factor_kernel' 0 tsqr
run l1err 'l1err_kernel' 0 l1err
