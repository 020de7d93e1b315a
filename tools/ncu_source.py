"""Per-kernel stall breakdown + hottest SASS lines from an ncu report (source page)."""
import csv
import subprocess
import sys


def main(rep, regex, top=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{regex}"], capture_output=True, text=True).stdout
    blocks, cur = [], None
    for l in out.split("\n"):
        if l.startswith('"Kernel Name"'):
            cur = [l]
            blocks.append(cur)
        elif cur is not None:
            cur.append(l)
    seen = set()
    for b in blocks:
        rows = list(csv.reader(b))
        name = rows[0][1][:70]
        if name in seen:
            continue
        seen.add(name)
        hdr = rows[1]
        si, samp = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
        cols = [c for c in hdr if c.startswith("stall_") and "(Not" not in c]
        data = []
        for r in rows[2:]:
            if len(r) < len(hdr):
                continue
            data.append((float(r[samp]), r[si].strip()[:80], {c: float(r[hdr.index(c)]) for c in cols}))
        tot = sum(d[0] for d in data) or 1
        agg = {c: sum(d[2][c] for d in data) for c in cols}
        print("=====", name, "samples", int(tot))
        print({k: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:7]})
        for v, s, st in sorted(data, key=lambda x: -x[0])[:top]:
            print(f"{100 * v / tot:5.1f}% {max(st, key=st.get):18s} {s}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 12)
