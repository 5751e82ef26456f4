"""Top source lines by warp-stall samples from an ncu report (--import-source on):
    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [launch_skip] [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      f"regex:{kre}", "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
fname, rows, tot = "?", [], 0.0
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif len(r) > 5 and r[0] not in ("", "Line No"):
        try:
            s = float(r[4])
        except ValueError:
            continue
        rows.append((s, fname, r[0], r[1].strip()))
        tot += s
rows.sort(key=lambda x: -x[0])
print(f"total samples {tot:.0f}")
for s, f, ln, src in rows[:top]:
    print(f"{100 * s / max(tot, 1):5.1f}% {f}:{ln:5s} {src[:100]}")
