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
REGEX = "regex:gemm_bf16_pair"
COUNT = 12          # the first GEMM launches of the step: several grouped-FFN pairs
rep = os.path.join(OUT, "ffn_pair")
cmd = ["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on",
       "--profile-from-start", "off", "--kernel-name-base", "demangled", "-k", REGEX, "-c", str(COUNT),
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
            "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}[u]


kernels = []
for r in data:
    rd = col("dram__bytes_read.sum", r) * scale("dram__bytes_read.sum")
    wr = col("dram__bytes_write.sum", r) * scale("dram__bytes_write.sum")
    t = col("gpu__time_duration.sum", r) * scale("gpu__time_duration.sum")
    kernels.append({"kernel": r[hdr.index("Kernel Name")], "dram_read_bytes": rd,
                    "dram_write_bytes": wr, "duration_s": t,
                    "tensor_pipe_pct": col("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", r)
                    if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed" in hdr else None})
import re  # noqa: E402


def shape(name):
    m = re.search(r"gemm_bf16_pair<(\d+), (\d+),", name)
    return (int(m.group(1)), int(m.group(2))) if m else None


# grouped-FFN pairs: the expert GEMM1 (256-wide tiles, GELU) directly followed by
# the expert GEMM2 with the pair-row epilogue (EPI_STORE_PAIR = 5)
pairs = [(a, b) for a, b in zip(kernels, kernels[1:])
         if shape(a["kernel"]) == (256, 1) and shape(b["kernel"]) == (192, 5)]
assert pairs, [k["kernel"] for k in kernels]
per_pair = [a["dram_read_bytes"] + a["dram_write_bytes"] + b["dram_read_bytes"]
            + b["dram_write_bytes"] for a, b in pairs]
total = sum(per_pair) / len(per_pair)
res = {"config": "xl256", "csrc_sha": bench.csrc_digest(),
       "traffic_bytes_per_launch_pair": total,
       "capture": (f"ncu --set full --clock-control none (cold caches): the first {COUNT} GEMM "
                   f"launches of step 7 of the bench workload (tools/profile_kernels.py); mean "
                   f"DRAM bytes over its {len(pairs)} grouped-FFN launch pairs"),
       "per_pair_bytes": per_pair,
       "kernels": kernels}
# gpurun brings back gpurun_out/ only: copy OUT/roofline_traffic.json to profiles/
with open(os.path.join(OUT, "roofline_traffic.json"), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
