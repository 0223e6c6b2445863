"""One warm XL async step (step 7 of the DICE schedule) bracketed by
cudaProfilerStart/Stop, for `ncu --set full --profile-from-start off -k ...`."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2411_16786_b200 as D

cfg = D.preset("xl2-8e2a", batch=32, num_steps=8)
model = D.init_model(cfg, seed=0)
x0 = D.sample_x0(cfg, 1000)
r = D.DeviceRunner(model, x0, D.Strategy.INTERWEAVED, D.dice_policy(), D.ClusterConfig(num_devices=1), 1000)
r.launch()
torch.cuda.synchronize()
r._reset_state()
for s in range(7):
    r._run_step(s)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r._run_step(7)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
