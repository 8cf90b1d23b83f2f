"""Summarise an ncu --set full report into profiles/: per-kernel duration,
DRAM bytes, tensor / XU pipe utilisation, registers, smem conflicts; and
update profiles/ncu_traffic.json (config:kernel -> DRAM bytes per launch),
which bench.py reports as roofline.traffic.

    python scripts/ncu_summary.py gpurun_out/prof_C3_r1.ncu-rep C3 r1
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1.0),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1.0),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1e6, "us": 1e3, "ns": 1,
              "usecond": 1e3, "msecond": 1e6, "nsecond": 1, "Ghz": 1, "Mhz": 1e-3, "hz": 1e-9}
NAMES = {"fwd_kernel": "fwd", "bwd_pre_kernel": "bwd_pre", "bwd_dkdv_kernel": "bwd_dkdv", "bwd_dq_kernel": "bwd_dq",
         "bwd_dqds_kernel": "bwd_dq_ds", "dq_convert_kernel": "dq_convert"}


def short_name(name):
    """bench.py's kernel names: bwd_dkdv_kernel<D, CAUSAL, FQ, DS> is bwd_dkdv_dq when fused (d = 64),
    bwd_dkdv_ds when it stores dS, bwd_dkdv otherwise."""
    short = next((v for k, v in NAMES.items() if k in name), None)
    if short == "bwd_dkdv":
        args = [a.strip() for a in name.split("<", 1)[1].split(">", 1)[0].split(",")]
        flags = [a.endswith("1") or a.endswith("true") for a in args[2:]]
        if flags and flags[0]:
            return "bwd_dkdv_dq"
        if len(flags) > 1 and flags[1]:
            return "bwd_dkdv_ds"
    return short


def main(rep, config, tag):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in data:
        name = r[idx["Kernel Name"]]
        short = short_name(name)
        if short is None:
            continue
        rec = {"kernel": short, "signature": name}
        for key, (m, _) in METRICS.items():
            if m not in idx:
                continue
            val = r[idx[m]].replace(",", "")
            try:
                x = float(val)
            except ValueError:
                continue
            u = units[idx[m]]
            if key == "duration_ms":
                x = x * UNIT_SCALE.get(u, 1) / 1e6
            elif "bytes" in key:
                x = x * UNIT_SCALE.get(u, 1)
            elif key == "sm_clock_ghz":
                x = x * UNIT_SCALE.get(u, 1)
            rec[key] = round(x, 4)
        if "dram_read_bytes" in rec:
            rec["dram_bytes_per_launch"] = rec["dram_read_bytes"] + rec.get("dram_write_bytes", 0)
        out.append(rec)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    base = os.path.join(ROOT, "profiles", f"ncu_{config}_{tag}")
    json.dump(out, open(base + ".json", "w"), indent=1)
    with open(base + ".md", "w") as f:
        f.write(f"# ncu --set full --clock-control none, {config}, round tag {tag}\n\n")
        f.write(f"Source report: `{os.path.basename(rep)}` (gpurun_out/, not tracked). One launch per kernel.\n\n")
        cols = ["kernel", "duration_ms", "dram_bytes_per_launch", "tensor_pipe_active_pct", "xu_pipe_pct",
                "fma_pipe_pct", "alu_pipe_pct", "dram_throughput_pct", "registers", "smem_bank_conflicts",
                "sm_clock_ghz"]
        f.write("| " + " | ".join(cols) + " |\n|" + "---|" * len(cols) + "\n")
        for rec in out:
            f.write("| " + " | ".join(str(rec.get(c, "")) for c in cols) + " |\n")
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    for rec in out:
        if "dram_bytes_per_launch" in rec:
            traffic[f"{config}:{rec['kernel']}"] = rec["dram_bytes_per_launch"]
    json.dump(traffic, open(tp, "w"), indent=1, sort_keys=True)
    print(open(base + ".md").read())


def launches(csv_path, out_md):
    """Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel share."""
    txt = open(csv_path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    tot, per = 0.0, {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", "")) * UNIT_SCALE.get(r["Metric Unit"], 1) / 1e6
        k = r["Kernel Name"]
        short = short_name(k) or re.sub(r"\(.*", "", k)[:60]
        per.setdefault(short, [0, 0.0])
        per[short][0] += 1
        per[short][1] += v
        tot += v
    with open(out_md, "w") as f:
        f.write(f"# ncu launch list summary ({os.path.basename(csv_path)})\n\n"
                "`ncu --metrics gpu__time_duration.sum --clock-control none` over a 2-step bench run "
                "(cold-cache, serialised: compare shares, not absolutes).\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {k} | {n} | {t:.3f} | {t / tot:.3f} |\n")
    print(open(out_md).read())


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        main(*sys.argv[1:4])
