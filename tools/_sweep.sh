python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for g in 3 0; do
  DICE_GATE4=$g python bench.py --no-cpu --no-quality > gpurun_out/b.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('gate4=$g', round(d['value'],2), d['clocks'], {k: round(v['us_per_call'],1) for k,v in d['breakdown'].items()})"
done
