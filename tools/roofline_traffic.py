"""DRAM traffic of the bench's roofline kernel (the grouped expert FFN launch
pair: expert GEMM1 + GELU carrying the stage's shared GEMM1, then the expert
GEMM2 with its pair-row epilogue) from ONE `ncu --set full` capture of the
first such pair of an asynchronous step of the bench workload
(tools/profile_kernels.py, step 7), written to profiles/roofline_traffic.json
with the CUDA-source digest it was taken on (copy OUT/roofline_traffic.json
there) (bench.py only uses it while the
sources are unchanged). Run under gpurun on one GPU:

  python tools/roofline_traffic.py [OUTDIR]
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

OUT = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "traffic")
os.makedirs(OUT, exist_ok=True)
REGEX = r"regex:gemm_bf16_pair<\(int\)(256, \(int\)1|192, \(int\)5),"
rep = os.path.join(OUT, "ffn_pair")
cmd = ["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on",
       "--profile-from-start", "off", "--kernel-name-base", "demangled", "-k", REGEX, "-c", "2",
       "-f", "-o", rep, sys.executable, os.path.join(ROOT, "tools", "profile_kernels.py")]
subprocess.run(cmd, check=True, cwd=ROOT)
raw = subprocess.run(["ncu", "-i", rep + ".ncu-rep", "--page", "raw", "--csv"], check=True,
                     capture_output=True, text=True).stdout
with open(os.path.join(OUT, "ffn_pair_raw.csv"), "w") as f:
    f.write(raw)
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]


def col(name, r):
    return float(r[hdr.index(name)].replace(",", ""))


def scale(name):
    u = units[hdr.index(name)]
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
            "usecond": 1e-6, "msecond": 1e-3}.get(u, 1)


kernels = []
for r in data:
    rd = col("dram__bytes_read.sum", r) * scale("dram__bytes_read.sum")
    wr = col("dram__bytes_write.sum", r) * scale("dram__bytes_write.sum")
    t = col("gpu__time_duration.sum", r) * scale("gpu__time_duration.sum")
    kernels.append({"kernel": r[hdr.index("Kernel Name")], "dram_read_bytes": rd,
                    "dram_write_bytes": wr, "duration_s": t,
                    "tensor_pipe_pct": col("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", r)
                    if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed" in hdr else None})
assert len(kernels) == 2, kernels
total = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in kernels)
res = {"config": "xl256", "csrc_sha": bench.csrc_digest(),
       "traffic_bytes_per_launch_pair": total,
       "capture": ("ncu --set full --clock-control none (cold caches), first grouped-FFN launch "
                   "pair of step 7 of the bench workload (tools/profile_kernels.py)"),
       "kernels": kernels}
# gpurun brings back gpurun_out/ only: copy OUT/roofline_traffic.json to profiles/
with open(os.path.join(OUT, "roofline_traffic.json"), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
