"""Top source lines of an ncu source page (`ncu -i X --page source --csv
--print-source cuda,sass`) by stall samples, with the dominant stall reason.
usage: python tools/ncu_lines.py page.csv source.cu [top]   (diagnostic tool)"""
import collections
import csv
import sys


def main(path, srcfile, top=30):
    rows = list(csv.reader(open(path)))
    hdr, f, agg = None, None, collections.defaultdict(lambda: [0.0, 0.0, {}])
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if len(r) < 10 or r[2] != "-":
            continue
        try:
            ln, w, n = int(r[0]), float(r[4] or 0), float(r[7] or 0)
        except ValueError:
            continue
        a = agg[(f, ln)]
        a[0] += n
        a[1] += w
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
                try:
                    a[2][h[6:]] = a[2].get(h[6:], 0.0) + float(r[i] or 0)
                except ValueError:
                    pass
    tw = sum(v[1] for v in agg.values()) or 1
    tn = sum(v[0] for v in agg.values()) or 1
    src = open(srcfile).read().split("\n")
    name = srcfile.split("/")[-1]
    print(f"warp-instructions {tn:.0f}, stall samples {tw:.0f}")
    for (ff, ln), (n, w, rs) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        t = max(rs.items(), key=lambda x: x[1])[0] if rs else ""
        txt = src[ln - 1].strip()[:90] if ff == name and ln <= len(src) else ""
        print(f"{n / tn * 100:5.1f}%I {w / tw * 100:5.1f}%S {t:10s} {ff}:{ln} {txt}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
