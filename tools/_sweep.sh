for cfg in "DICE_GEMM_WIDE=1" "DICE_GEMM_WIDE=0" "DICE_GEMM_WIDE=0 DICE_GEMM_EPI_DIRECT=0"; do
  env $cfg python bench.py --no-cpu --no-quality > gpurun_out/b.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('$cfg', round(d['value'],2), round(d['roofline']['frac'],3), d['moe_layer_us'], d['clocks'])"
done
env DICE_GEMM_WIDE=1 python bench.py --no-cpu --no-quality --overlap > gpurun_out/b.log 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('overlap', round(d['value'],2), round(d['roofline']['frac'],3), d['moe_layer_us'], d['clocks'])"
