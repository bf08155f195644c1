"""Static SASS instruction count per source line of one kernel (nvdisasm -g
on the built object).  Diagnostic tool: code size drives instruction-cache
misses in the fused step+observe kernel.
usage: python tools/sass_lines.py [kernel-substring] [top]"""
import collections
import re
import subprocess
import sys
import tempfile
from pathlib import Path

EXCL = "--excl" in sys.argv  # count each instruction for its innermost line only
sys.argv = [a for a in sys.argv if a != "--excl"]
OBJ = Path(__file__).resolve().parent.parent / "paper_2312_15122_b200" / "_build" / (sys.argv[3] if len(sys.argv) > 3 else "") / "zsim_kernels.cu.o"


def main(sub="ILb1ELi3ELb0", top=40):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(OBJ)], cwd=d, check=True, capture_output=True)
        cub = next(Path(d).glob("*.cubin"))
        sass = subprocess.run(["nvdisasm", "-gi", str(cub)], capture_output=True, text=True).stdout
    # inclusive: an instruction counts for its line and every call site it is inlined at
    cnt, fn, chain, fresh = collections.Counter(), None, set(), False
    for l in sass.split("\n"):
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            fn = m.group(1)
            continue
        if "//## File" in l:
            if not fresh:
                chain, fresh = set(), True
            elif EXCL:
                continue
            for f, ln in re.findall(r'"([^"]+)", line (\d+)', l)[:1 if EXCL else None]:
                chain.add((f.split("/")[-1], int(ln)))
            continue
        if fn and sub in fn and re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
            fresh = False
            for c in chain:
                cnt[c] += 1
    src = {}
    for k, _ in cnt.most_common(top):
        if k and k[0] not in src:
            p = next((q for q in (OBJ.parent.parent / "csrc").glob(k[0])), None)
            src[k[0]] = p.read_text().split("\n") if p else []
    print("exclusive" if EXCL else "inclusive (call sites include their inlined callees)",
          "static SASS instructions per source line")
    for k, v in cnt.most_common(top):
        txt = src.get(k[0], [])[k[1] - 1].strip()[:80] if k and k[1] <= len(src.get(k[0], [])) else ""
        print(f"{v:6d} {k[0]}:{k[1]}  {txt}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "ILb1ELi3ELb0", int(sys.argv[2]) if len(sys.argv) > 2 else 40)
