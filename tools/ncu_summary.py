"""Summarise an ncu report (raw page) into the metrics we track.
usage: python tools/ncu_summary.py report.ncu-rep [--json out.json]"""
import csv, io, json, subprocess, sys

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "mufu_xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct": "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "registers": "launch__registers_per_thread",
}
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}

def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    outs = [_one(dict(zip(hdr, zip(units, vals)))) for vals in rows[2:]]
    return outs[0] if len(outs) == 1 else outs


def _one(d):
    out = {"kernel": d.get("Kernel Name", ("", ""))[1]}
    for k, m in KEYS.items():
        if m not in d:
            continue
        u, v = d[m]
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        if k.endswith("_bytes"):
            x *= UNIT.get(u, 1)
        if k == "duration_ms" and u == "usecond":
            x /= 1e3
        out[k] = x
    stalls = []
    for h, (u, v) in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    out["stall_top"] = {n: round(s / tot * 100, 1) for s, n in sorted(stalls, reverse=True)[:8]}
    return out

if __name__ == "__main__":
    s = summarise(sys.argv[1])
    print(json.dumps(s, indent=1))
    if "--json" in sys.argv:
        json.dump(s, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
