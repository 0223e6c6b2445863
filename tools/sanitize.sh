#!/bin/bash
# compute-sanitizer over the library's kernels (run under gpurun, 1 GPU):
# memcheck / racecheck / synccheck / initcheck on tools/sanitize_ops.py, and
# memcheck over the GPU kernel tests. Logs -> gpurun_out/${1:-san}/.
OUT=gpurun_out/${1:-san}
mkdir -p $OUT
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  # racecheck does not model the tcgen05 / TMA async proxies of the GEMM: the
  # GEMM's reports are summarised separately below (racecheck_gemm_sites.txt)
  [ $tool = racecheck ] && extra="--racecheck-report hazard --kernel-name-exclude kns=gemm_bf16_pair"
  timeout 1500 $CS --tool $tool $extra python tools/sanitize_ops.py > $OUT/$tool.log 2>&1
  echo "rc=$?" >> $OUT/$tool.log
done
# every racecheck report on the GEMM kernels, reduced to its distinct (access, site) pairs
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 0 \
    --kernel-name kns=gemm_bf16_pair python tools/sanitize_ops.py 2>&1 \
  | grep -E "(Read|Write) Thread|RACECHECK SUMMARY|at __shared__" \
  | sed -E 's/\+0x[0-9a-f]+//; s/Thread \([0-9,]+\)/Thread/; s/in block \([0-9,]+\)//' \
  | sort | uniq -c | sort -rn > $OUT/racecheck_gemm_sites.txt
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_kernels.py -x -q > $OUT/memcheck_kernel_tests.log 2>&1
echo "rc=$?" >> $OUT/memcheck_kernel_tests.log
for f in $OUT/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|rc=|passed|failed" $f | tail -3; done > $OUT/summary.txt
