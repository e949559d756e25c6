"""Hot source lines of one kernel in an ncu report (warp-stall samples per CUDA line).
Usage: python tools/ncu_hot_lines.py report.ncu-rep [kernel-substring] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
func, hdr, cur = None, None, None
acc = {}
for x in rows:
    if len(x) == 2 and x[0] == "Function Name":
        func = x[1]
        continue
    if len(x) > 4 and x[0] == "Line No":
        hdr = x
        continue
    if not hdr or len(x) != len(hdr) or want not in (func or ""):
        continue
    if x[0]:
        cur = (x[0], x[1][:110])
        try:
            acc[cur] = acc.get(cur, 0.0) + float(x[4])
        except ValueError:
            pass
tot = sum(acc.values()) or 1.0
for (line, src), v in sorted(acc.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v / tot * 100:5.1f}%  L{line:>4}  {src.strip()}")
