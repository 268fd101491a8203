"""Hot SASS regions of one kernel from `ncu --page source --csv --print-source sass`
output: consecutive instructions with equal execution counts are grouped
(basic-block approximation) and ranked by executed warp instructions."""
import csv
import sys


def main(path, which=0, top=25):
    rows = list(csv.reader(open(path)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    a = starts[which]
    b = starts[which + 1] if which + 1 < len(starts) else len(rows)
    print(rows[a][1][:100])
    h = rows[a + 1]
    data = [r for r in rows[a + 2:b] if len(r) == len(h)]
    si, ei = h.index("Source"), h.index("Instructions Executed")
    wi = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[ei]) for r in data)
    samp = max(1, sum(int(r[wi]) for r in data))
    segs, cur = [], None
    for idx, r in enumerate(data):
        c = int(r[ei])
        if cur and cur["c"] == c:
            cur["n"] += 1
            cur["end"] = idx
            cur["s"] += int(r[wi])
        else:
            cur = {"c": c, "start": idx, "end": idx, "n": 1, "s": int(r[wi])}
            segs.append(cur)
    segs.sort(key=lambda s: -s["c"] * s["n"])
    acc = 0
    print("total warp instructions", tot)
    for s in segs[:top]:
        w = s["c"] * s["n"]
        acc += w
        ops = {}
        for r in data[s["start"]:s["end"] + 1]:
            t = r[si].split()
            op = t[1] if t[0].startswith("@") else t[0]
            op = op.split(".")[0]
            ops[op] = ops.get(op, 0) + 1
        topo = sorted(ops.items(), key=lambda x: -x[1])[:6]
        print(f"{s['start']:5d}-{s['end']:5d} n={s['n']:4d} exec={s['c']:9d} share={w / tot * 100:5.1f}% "
              f"cum={acc / tot * 100:5.1f}% stall={s['s'] / samp * 100:4.1f}% {topo}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
