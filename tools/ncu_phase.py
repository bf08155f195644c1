"""Aggregate an ncu source page (`ncu -i X --page source --csv --print-source cuda,sass`)
by enclosing function of zsim_kernels.cu, using the source text embedded in the
report (so line numbers match the profiled build).  Diagnostic tool."""
import csv
import re
import sys
from pathlib import Path

KSRC = Path(__file__).resolve().parent.parent / "paper_2312_15122_b200" / "csrc" / "zsim_kernels.cu"


def main(path, top=0):
    rows = list(csv.reader(open(path)))
    lines = {}  # (file, line) -> (inst, samples, text, {stall reason: samples})
    f = None
    hdr = None
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
            n, w, ln = float(r[7] or 0), float(r[4] or 0), int(r[0])
        except ValueError:
            continue
        a = lines.setdefault((f, ln), [0.0, 0.0, r[1], {}])
        a[0] += n
        a[1] += w
        if hdr:
            for i, h in enumerate(hdr):
                if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
                    try:
                        a[3][h[6:]] = a[3].get(h[6:], 0.0) + float(r[i] or 0)
                    except ValueError:
                        pass
    # function ranges from the current source; profiled lines are matched to it
    # by text (nearest identical line), so edits since the capture do not shift them
    src = open(KSRC).read().split("\n")
    starts = []
    for i, txt in enumerate(src, 1):
        m = re.match(r"\s*(?:__device__|__global__)[^(]*?(\w+)\(", txt)
        if m and "#define" not in txt:
            starts.append((i, m.group(1)))
    by_text = {}
    for i, txt in enumerate(src, 1):
        by_text.setdefault(txt.strip(), []).append(i)

    def cur_line(ln, txt):
        c = by_text.get(txt.strip())
        return min(c, key=lambda i: abs(i - ln)) if c else ln

    agg = {}
    reasons = {}
    for (ff, ln), (n, w, txt, rs) in lines.items():
        key = ff
        if ff == "zsim_kernels.cu":
            key = "?"
            cl = cur_line(ln, txt)
            for s, nm in starts:
                if s <= cl:
                    key = nm
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += n
        a[1] += w
        rr = reasons.setdefault(key, {})
        for k, v in rs.items():
            rr[k] = rr.get(k, 0.0) + v
    tot = sum(v[0] for v in agg.values()) or 1
    totw = sum(v[1] for v in agg.values()) or 1
    print(f"total warp-instructions {tot:.0f}, stall samples {totw:.0f}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        rtop = sorted(reasons.get(k, {}).items(), key=lambda x: -x[1])[:4]
        ts = " ".join(f"{a}:{b / max(v[1], 1) * 100:.0f}%" for a, b in rtop if b > 0)
        print(f"{k:28s} inst {v[0] / tot * 100:5.1f}%  stall-samples {v[1] / totw * 100:5.1f}%  [{ts}]")
    if top:
        print("--- top lines by stall samples")
        for (ff, ln), (n, w, txt, rs) in sorted(lines.items(), key=lambda x: -x[1][1])[:top]:
            tr = max(rs.items(), key=lambda x: x[1])[0] if rs else ""
            print(f"{n / tot * 100:5.1f}%I {w / totw * 100:5.1f}%S {tr[:9]:9s} {ff[:16]}:{ln:>4} {txt.strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
