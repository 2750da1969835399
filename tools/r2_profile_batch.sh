#!/bin/bash
# Round-2 profile batch (run under gpurun): ncu --set full of the dominant Ozaki GEMM shape and of the
# warp-sliced Jacobi SVD, the launch list of one matvec+round step, and the same-config (mode size
# 1024) host timing of the reference algorithm (bench.py --impl reference).
set -u
mkdir -p gpurun_out
python tools/ncu_ozaki.py 1048576 1024 1024 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
  -k "regex:oz_gemm_kernel" --launch-count 1 -o gpurun_out/r2_ncu_full_ozaki_1m_1k_1k -f \
  python tools/ncu_ozaki.py 1048576 1024 1024 > gpurun_out/ncu_oz.log 2>&1; echo "ozaki ncu $?"
python tools/one_svd.py > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:jacobi_wslice" --launch-count 1 \
  -o gpurun_out/r2_ncu_full_jacobi_wslice -f python tools/one_svd.py > gpurun_out/ncu_jw.log 2>&1; echo "jacobi ncu $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/r2_launches_matvec_round.csv python bench.py --steps 1 --warmup 1 --skip-solve --skip-cpu \
  --skip-dmma > gpurun_out/ncu_launch.log 2>&1; echo "launch list $?"
free -g | head -2; nproc
timeout 1200 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2_reference_arm_n1024.log 2>&1; echo "ref arm $?"
