for cfg in "DICE_SHARED_SPLIT=2" "DICE_SHARED_SPLIT=1" "DICE_SHARED_SPLIT=4"; do
  env DICE_MERGE_GEMM1=0 DICE_MERGE_THEN=0 $cfg python bench.py --no-cpu --no-quality > gpurun_out/b.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('$cfg', round(d['value'],2), d['clocks']['sm_mhz'], {k: round(v['us_per_call'],1) for k,v in d['breakdown'].items()})"
done
nvidia-smi --query-gpu=power.draw,power.limit,clocks.sm --format=csv
