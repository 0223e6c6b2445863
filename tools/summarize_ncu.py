"""Summarise ncu --set full CSV exports (tools/profile_round.sh) into one text
table: per kernel the duration, DRAM bytes, throughputs, tensor-pipe share,
occupancy and registers. python tools/summarize_ncu.py DIR > summary.txt"""
import csv
import glob
import os
import sys

d = sys.argv[1]
KEYS = [("gpu__time_duration.sum", "duration us"), ("dram__bytes_read.sum", "DRAM read MB"),
        ("dram__bytes_write.sum", "DRAM write MB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
        ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "L2 sectors % of peak"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % active"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
        ("launch__registers_per_thread", "registers/thread"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("sm__cycles_elapsed.avg.per_second", "SM clock GHz")]
for path in sorted(glob.glob(os.path.join(d, "k*_raw.csv"))):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        continue
    h, units, v = rows[0], rows[1], rows[2]
    print(v[h.index("Kernel Name")])
    for key, label in KEYS:
        if key in h:
            i = h.index(key)
            print(f"    {label:26s} {v[i]:>14s} {units[i]}")
    print()
