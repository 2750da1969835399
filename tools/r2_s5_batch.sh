#!/bin/bash
# Round-2 (session 5) batch under gpurun: rounding tests, a short bench line, and ncu --set full of the
# 1024 x 1048576 x 1024 Ozaki GEMM (the left-to-right carry of the matvec+round step).
set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_matvec_round.py tests/test_gpu_host.py tests/test_gpu_kernels.py -x -q -s > gpurun_out/s5_tests_round.log 2>&1; echo "tests $?"
tail -3 gpurun_out/s5_tests_round.log
python bench.py --skip-solve --skip-cpu > gpurun_out/s5_bench_short.log 2> gpurun_out/s5_bench_short.err; echo "bench $?"
python tools/ncu_ozaki.py 1024 1048576 1024 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" \
  -k "regex:oz_gemm_kernel" --launch-count 1 -o gpurun_out/r2_ncu_full_ozaki_1k_1m_1k -f \
  python tools/ncu_ozaki.py 1024 1048576 1024 > gpurun_out/ncu_oz2.log 2>&1; echo "ozaki ncu $?"
