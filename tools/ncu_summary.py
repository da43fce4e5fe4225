"""Turn ncu raw-page CSV exports into profiles/ncu_summary.json + a markdown table.

    python tools/ncu_summary.py profiles/r1/ncu_raw_dvr_cfg2.csv:cfg2 profiles/r1/ncu_raw_decode_cfg4.csv:cfg4
"""
import csv
import json
import sys
from pathlib import Path

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "instructions": ("smsp__inst_executed.sum", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    "lsu_pipe_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "sm_ghz": ("sm__cycles_elapsed.avg.per_second", 1),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6,
        "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1}


def parse(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, zip(units, vals)))
    out = {"kernel": d.get("Kernel Name", ("", ""))[1]}
    stalls = {}
    for k, (metric, scale) in KEYS.items():
        if metric not in d:
            continue
        u, v = d[metric]
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        if k == "duration_ms":
            x *= UNIT.get(u, 1) if u in ("ns", "nsecond", "us", "usecond", "ms", "msecond") else 1
        elif scale is None:
            x *= UNIT.get(u, 1)
        out[k] = x
    for h, (u, v) in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
    out["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    out["dram_bytes_per_launch"] = out.get("dram_read_bytes", 0) + out.get("dram_write_bytes", 0)
    return out


def main():
    summary = {}
    dst = Path("profiles/ncu_summary.json")
    if dst.exists():
        summary = json.loads(dst.read_text())
    for arg in sys.argv[1:]:
        path, cfg = arg.rsplit(":", 1)
        summary[cfg] = {"source": path, **parse(path)}
    dst.write_text(json.dumps(summary, indent=1))
    for cfg, s in summary.items():
        print(f"## {cfg}: {s['kernel'][:60]}")
        for k in KEYS:
            if k in s:
                print(f"  {k:20s} {s[k]}")
        print(f"  top stalls: {s['top_stalls_per_issue']}")


if __name__ == "__main__":
    main()
