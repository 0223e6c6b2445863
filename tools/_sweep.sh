for f in 1 0; do
  DICE_MERGE_GEMM1=$f python bench.py --no-cpu --no-quality > gpurun_out/b.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('merge=$f', round(d['value'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), {k: round(v['us_per_call'],1) for k,v in d['breakdown'].items()})"
done
