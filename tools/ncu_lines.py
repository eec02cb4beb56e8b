"""Per-CUDA-source-line executed warp instructions + stall samples of an ncu
report (needs -lineinfo and --import-source on).  Usage: ncu_lines.py rep [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, lines, tot, stot = None, [], 0, 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 10 or r[0] == "Line No" or not r[0].isdigit():
        continue
    try:
        ie, ss = int(r[7]), int(r[4])
    except ValueError:
        continue
    tot += ie; stot += ss
    lines.append((ie, ss, fname, int(r[0]), r[1].strip()[:90]))
print(f"total warp-instr {tot}  stall samples {stot}")
for ie, ss, f, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100*ie/tot:5.1f}% {100*ss/max(stot,1):5.1f}%s {f}:{ln:5d} {src}")
