#!/bin/bash
# Round profile capture (run under gpurun, 1 GPU): launch list of the bench
# workload's steps 6-7 (the recipe's cold-cache pass) + one ncu --set full
# launch of each top kernel of an async step (7). CSV exports only (small).
OUT=gpurun_out/${1:-prof}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $OUT/launches_steps6-7.csv python tools/profile_step.py > $OUT/launch.log 2>&1
python tools/summarize_launches.py $OUT/launches_steps6-7.csv > $OUT/launch_summary.txt
i=0
for k in "gemm_bf16_pair<.int.256, .int.1," "gemm_bf16_pair<.int.192, .int.4," \
         "gemm_bf16_pair<.int.192, .int.5," "gemm_bf16_pair<.int.192, .int.3," "gate4_topk"; do
  i=$((i+1))
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
      --kernel-name-base demangled -k "regex:$k" -s 1 -c 1 -o $OUT/k$i python tools/profile_kernels.py \
      > $OUT/k$i.log 2>&1
  ncu -i $OUT/k$i.ncu-rep --page raw --csv > $OUT/k${i}_raw.csv 2>/dev/null
  ncu -i $OUT/k$i.ncu-rep --page details --csv > $OUT/k${i}_details.csv 2>/dev/null
  if [ $i -ge 5 ]; then   # memory-bound kernels: keep the source-level view
    ncu -i $OUT/k$i.ncu-rep --page source --csv --print-source sass > $OUT/k${i}_sass.csv 2>/dev/null
  fi
  rm -f $OUT/k$i.ncu-rep
done
python tools/summarize_ncu.py $OUT > $OUT/ncu_summary.txt
du -sh $OUT
