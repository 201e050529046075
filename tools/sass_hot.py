"""Hot SASS of one kernel from an ncu report (development tool):
    python tools/sass_hot.py REPORT.ncu-rep KERNEL_REGEX [N]
prints total executed warp-instructions, stall-sample totals by reason, and
the N hottest instructions (executed count, stall samples)."""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{rx}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) == len(h)]
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
tot = sum(int(r[ie] or 0) for r in body)
print(f"instructions: {len(body)} static, {tot} executed (warp)")
st = {h[i]: sum(int(r[i] or 0) for r in body) for i in stall_cols}
print("stall samples:", {k: v for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v})
body2 = sorted(enumerate(body), key=lambda kv: -int(kv[1][ie] or 0))[:N]
for idx, r in sorted(body2):
    print(f"{idx:5d} {int(r[ie]):>11d} {int(r[ss] or 0):>6d}  {r[1].strip()}")

# execution-count histogram: static instructions per distinct count (loop bodies)
from collections import Counter
cnt = Counter(int(r[ie] or 0) for r in body)
print("executed-count -> static instrs (top by executed total):")
for c, k in sorted(cnt.items(), key=lambda kv: -kv[0] * kv[1])[:15]:
    print(f"  {c:>11d} x {k:4d} = {c * k:>12d}")
