"""Per-instruction stall samples of an ncu report (--set full, -lineinfo):
python tools/sass_hot.py REPORT KERNEL_REGEX [N]."""
import csv
import subprocess
import sys
from collections import Counter


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main(rep, kern, n=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]
    si, ns, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index(
        "Instructions Executed")
    tot = sum(num(r[ns]) for r in data)
    print("total samples", tot, "instructions", sum(num(r[ie]) for r in data))
    c, ci = Counter(), Counter()
    for r in data:
        t = r[si].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        op = op.split(".")[0]
        c[op] += num(r[ns])
        ci[op] += num(r[ie])
    for k, v in c.most_common(20):
        print(f"{k:12s} samples {v:7d} {100 * v / max(tot, 1):5.1f}%  instr {ci[k]}")
    cols = [x for x in ("stall_wait", "stall_short_sb", "stall_long_sb", "stall_mio", "stall_math",
                        "stall_lg", "stall_barrier", "stall_branch_resolving", "stall_no_inst")
            if x in h]
    cix = [h.index(x) for x in cols]
    print("cols:", cols)
    for i in sorted(sorted(range(len(data)), key=lambda i: -num(data[i][ns]))[:n]):
        r = data[i]
        print(f"{i:5d} {r[si].strip()[:58]:58s} {num(r[ns]):6d}", [num(r[j]) for j in cix])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
