"""Summarise an ncu --set full report (one kernel launch) into JSON: duration, DRAM bytes
read/written, throughput, occupancy, issue activity; with --step (tools/profile_step.py
output) also the algorithmic bytes of that launch and the traffic / algorithmic ratio.
Usage: python tools/ncu_summary.py report.ncu-rep [--step step.json] [--out summary.json]"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__inst_executed.sum": "inst_executed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")}
        for k, name in KEYS.items():
            v = d.get(k)
            if v not in (None, ""):
                try:
                    rec[name] = float(v.replace(",", "")) * scale.get(units.get(k, ""), 1.0)
                except ValueError:
                    rec[name] = v
        out.append(rec)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--step")
    ap.add_argument("--out")
    a = ap.parse_args()
    launches = raw(a.report)
    summary = {"report": a.report, "launches": launches}
    if a.step:
        st = json.load(open(a.step))
        summary["step"] = st
        for rec in launches:
            kn = rec["kernel"]
            key = "policy" if "k_policy" in kn else "hh" if "k_prepare_p" in kn else "post" if "k_post" in kn else None
            if key and f"{key}_algorithmic_bytes" in st:
                traffic = rec.get("dram_read_bytes", 0) + rec.get("dram_write_bytes", 0)
                alg = st[f"{key}_algorithmic_bytes"]
                rec["algorithmic_bytes"] = alg
                rec["traffic_over_algorithmic"] = traffic / alg
                rec["algorithmic_GBps"] = alg / rec["duration_ns"]
    txt = json.dumps(summary, indent=1)
    if a.out:
        open(a.out, "w").write(txt)
    print(txt)
