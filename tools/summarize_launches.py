"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel count/total and the per-evaluate launch sequence."""
import csv
import sys


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    gi, bi = hdr.index("Grid Size"), hdr.index("Block Size")
    seq = [(r[ki].split("(")[0].split("::")[-1].replace("void ", ""), r[gi], r[bi],
            float(r[vi].replace(",", "")) / 1e3) for r in rows[1:]]
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    agg = {}
    for k, _, _, t in seq:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    starts = [i for i, s in enumerate(seq) if s[0].startswith(("gather_charges", "gather_pack"))]
    if len(starts) >= 2:
        lines += ["", "One evaluate (second in the run), in launch order:", "",
                  "| kernel | grid | block | us |", "|---|---|---|---|"]
        end = starts[2] if len(starts) > 2 else len(seq)
        for k, g, b, t in seq[starts[1]:end]:
            lines.append(f"| {k} | {g} | {b} | {t:.1f} |")
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
