for cfg in "DICE_GEMM_CHAIN=1" "DICE_GEMM_CHAIN=2" "DICE_GEMM_WIDE=1"; do
  env $cfg python bench.py --no-cpu --no-quality > gpurun_out/b.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('$cfg', round(d['value'],2), d['clocks']['sm_mhz'], {k: round(v['us_per_call'],1) for k,v in d['breakdown'].items()})"
done
