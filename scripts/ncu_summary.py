"""Summarise `ncu --set full` reports (gpurun_out/*.ncu-rep) into profiles/: one
text block per kernel with the metrics the roofline and DESIGN.md cite, and
profiles/traffic.json (dram read+write bytes per launch, read by bench.py)."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum"]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        m = {k: (d[k], units[h.index(k)]) for k in KEYS if k in d}
        res.append((d["Kernel Name"], m))
    return res


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]


if __name__ == "__main__":
    outdir, config, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    traffic_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for rep in reps:
        name = os.path.basename(rep).replace(".ncu-rep", "")
        lines = []
        for kern, m in summarise(rep):
            lines.append(f"kernel: {kern}")
            for k, (v, u) in m.items():
                lines.append(f"  {k:62s} {v} {u}")
            if "dram__bytes_read.sum" in m:
                t = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
                lines.append(f"  traffic (dram read+write) per launch: {t:.6g} B")
                short = kern.split("(")[0].split("<")[0].replace("void ", "").strip()
                traffic.setdefault(config, {})[short] = t
        open(os.path.join(outdir, f"ncu_{name}.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    json.dump(traffic, open(traffic_path, "w"), indent=1)
