"""Executed SASS instruction mix (+ stall samples) of an ncu report."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
isrc, iex, iss = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
cnt, st, tot = collections.Counter(), collections.Counter(), 0
hot = []
for r in rows[2:]:
    try:
        n, s = int(r[iex]), int(r[iss])
    except ValueError:
        continue
    op = r[isrc].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    cnt[o.split(".")[0]] += n
    st[o.split(".")[0]] += s
    tot += n
    hot.append((s, r[isrc].strip()[:70]))
print("total warp-instr", tot)
for o, n in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{o:10s} {n:12d} {100*n/tot:5.1f}%  stall-samples {st[o]}")
print("hottest:")
for s, src in sorted(hot, reverse=True)[:12]:
    print(f"{s:7d}  {src}")
