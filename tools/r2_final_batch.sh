#!/bin/bash
# Round-2 evidence batch (run under gpurun): the full GPU suite, the default bench line, the reference arm
# at the bench's own arguments, and the ncu launch list of one matvec+round step.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -s > gpurun_out/r2_gputest.log 2>&1; echo "tests $?"; tail -2 gpurun_out/r2_gputest.log
if [ -d tools/refsuite/tests ]; then   # the reference's own suite against this package (tools/refsuite/fetch.py)
  (cd tools/refsuite && python -m pytest tests -q -p no:cacheprovider --ignore=tests/test_cli.py > ../../gpurun_out/r2_refsuite.log 2>&1); echo "refsuite $?"; tail -1 gpurun_out/r2_refsuite.log
fi
python bench.py > gpurun_out/r2_bench_full.log 2> gpurun_out/r2_bench_full.err; echo "bench $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/r2_launches_matvec_round.csv python bench.py --steps 1 --warmup 1 --skip-solve --skip-cpu \
  --skip-dmma > gpurun_out/ncu_launch.log 2>&1; echo "launch list $?"
