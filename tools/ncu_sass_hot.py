"""Top SASS lines by warp-stall samples from an ncu report.
usage: python tools/ncu_sass_hot.py report.ncu-rep kernel_regex [N]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
val = lambda r: float(r[i_s] or 0)  # noqa: E731
tot = sum(val(r) for r in data) or 1
for idx, r in sorted(enumerate(data), key=lambda x: -val(x[1]))[:n]:
    print(f"{val(r) / tot * 100:5.1f}%  #{idx:5d}  {r[1].strip()[:100]}")
