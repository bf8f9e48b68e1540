"""Summarise ncu `--page raw --csv` exports (gpurun_out/prof/*.raw.csv, written by
scripts/gpu_profiles_r02.sh) into profiles/r02/ncu_<tag>.txt, the launch lists into
profiles/r02/launches_<config>.txt, and refresh profiles/traffic.json (dram read + write bytes
per launch of the dominant sweep, with the capture it came from)."""
import collections
import csv
import glob
import io
import json
import os
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum"]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main(src, out):
    os.makedirs(out, exist_ok=True)
    traffic = {}
    for f in sorted(glob.glob(os.path.join(src, "*.raw.csv"))):
        tag = os.path.basename(f)[: -len(".raw.csv")]
        rows = list(csv.reader(open(f)))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        d = dict(zip(h, rows[2]))
        lines = [f"kernel: {d.get('Kernel Name', '?')}", f"capture: {tag} (ncu --set full --clock-control none, "
                 "one launch of the second retrieval, scripts/gpu_profiles_r02.sh)"]
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:<66} {d[k]} {units[h.index(k)]}")
        rb = to_bytes(d["dram__bytes_read.sum"], units[h.index("dram__bytes_read.sum")])
        wb = to_bytes(d["dram__bytes_write.sum"], units[h.index("dram__bytes_write.sum")])
        lines.append(f"  traffic (dram read + write) per launch: {rb + wb:.6g} B")
        open(os.path.join(out, f"ncu_{tag}.txt"), "w").write("\n".join(lines) + "\n")
        traffic[tag] = rb + wb
    for f in sorted(glob.glob(os.path.join(src, "launches_*.csv"))):
        cfg = os.path.basename(f)[len("launches_"):-4]
        txt = open(f).read()
        body = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
        rows = list(csv.reader(io.StringIO(body)))
        h = rows[0]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        agg = collections.OrderedDict()
        for r in rows[1:]:
            if len(r) <= vi:
                continue
            name = r[ki].split("(")[0]
            n, t = agg.get(name, (0, 0.0))
            agg[name] = (n + 1, t + float(r[vi].replace(",", "")))
        tot = sum(t for _, t in agg.values())
        lines = [f"launch list, {cfg}: two retrievals (warm-up + measured), ncu gpu__time_duration.sum "
                 "--clock-control none (cold-cache, serialised: compare shares, not absolutes)",
                 f"{'kernel':<40} {'launches':>8} {'total us':>12} {'avg us':>10} {'share':>7}"]
        for name, (n, t) in agg.items():
            lines.append(f"{name:<40} {n:>8} {t / 1e3:>12.1f} {t / n / 1e3:>10.2f} {t / tot:>7.3f}")
        open(os.path.join(out, f"launches_{cfg}.txt"), "w").write("\n".join(lines) + "\n")
    tjp = os.path.join(os.path.dirname(out.rstrip("/")), "traffic.json")
    tj = json.load(open(tjp)) if os.path.exists(tjp) else {}   # merge: a partial capture set keeps the rest
    if "fl_k3" in traffic:
        tj["flightline"] = {"k3_sweep": traffic["fl_k3"], "source": "profiles/r02/ncu_fl_k3.txt"}
    if "st_k3w" in traffic:
        tj["stress"] = {"k3_sweep": traffic["st_k3w"], "source": "profiles/r02/ncu_st_k3w.txt"}
    json.dump(tj, open(os.path.join(os.path.dirname(out.rstrip("/")), "traffic.json"), "w"), indent=1)
    print("wrote", out, sorted(traffic))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof", sys.argv[2] if len(sys.argv) > 2 else "profiles/r02")
