"""Summarise ncu reports (gpurun_out/*.ncu-rep) into profiles/: key metrics per
kernel and profiles/ncu_traffic.json (dram bytes per launch) for bench.py."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "launch__shared_mem_per_block_dynamic": "smem_dyn",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    val = float(v) * UNIT.get(units[i], 1)
                except ValueError:
                    val = v
                d[name] = val
        res.append(d)
    return res


def main(tag, reps):
    summary, traffic = {}, {}
    for op, rep in reps.items():
        r = read(rep)
        if not r:
            continue
        d = r[0]
        summary[op] = d
        traffic[op] = int(d.get("dram_read", 0) + d.get("dram_write", 0))
    os.makedirs("profiles", exist_ok=True)
    with open(f"profiles/{tag}_ncu_full_summary.json", "w") as f:
        json.dump(summary, f, indent=1)
    with open("profiles/ncu_traffic.json", "w") as f:
        json.dump(traffic, f, indent=1)
    for op, d in summary.items():
        print(op, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items() if k != "kernel"}, d["kernel"][:60])


if __name__ == "__main__":
    tag = sys.argv[1]
    reps = {}
    for fn in sorted(os.listdir("gpurun_out")):
        if fn.startswith(f"{tag}_full_") and fn.endswith(".ncu-rep"):
            reps[fn[len(tag) + 6:-8]] = os.path.join("gpurun_out", fn)
    main(tag, reps)
