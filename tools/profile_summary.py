"""Summarise one bench + ncu round trip (gpurun_out/) into profiles/<tag>_*.

    python tools/profile_summary.py <tag>

Reads gpurun_out/bench_line.json, gpurun_out/launches.csv (ncu launch list)
and gpurun_out/prof_bench.ncu-rep (ncu --set full of k_step_observe); writes
profiles/<tag>_bench.json, <tag>_launches.csv, <tag>_ncu_full.csv,
<tag>_summary.md and refreshes profiles/ncu_traffic.json.  Diagnostic tool.
"""
import csv
import io
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local ld sectors"),
    ("l1tex__t_sector_pipe_lsu_mem_local_op_ld_hit_rate.pct", "local ld L1 hit %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard / issue"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def ncu_raw(rep: Path) -> dict:
    r = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    return {h: (rows[2][i], rows[1][i]) for i, h in enumerate(rows[0])}


def main(tag: str) -> None:
    line = json.loads((OUT / "bench_line.json").read_text())
    (PROF / f"{tag}_bench.json").write_text(json.dumps(line, indent=1) + "\n")
    shutil.copy(OUT / "launches.csv", PROF / f"{tag}_launches.csv")
    txt = (OUT / "launches.csv").read_text().splitlines()
    i = next(k for k, l in enumerate(txt) if l.startswith('"ID"'))
    per = defaultdict(list)
    for x in csv.DictReader(io.StringIO("\n".join(txt[i:]))):
        per[x["Kernel Name"].split("(")[0][:48]].append(float(x["Metric Value"]))
    tot = sum(sum(v) for v in per.values())
    rep = OUT / "prof_bench.ncu-rep"
    r = subprocess.run(["ncu", "-i", str(rep), "--page", "details", "--csv"], capture_output=True, text=True)
    (PROF / f"{tag}_ncu_full.csv").write_text(r.stdout)
    raw = ncu_raw(rep)
    rd = float(raw["dram__bytes_read.sum"][0]) * (1e6 if raw["dram__bytes_read.sum"][1].startswith("M") else 1)
    wr = float(raw["dram__bytes_write.sum"][0]) * (1e6 if raw["dram__bytes_write.sum"][1].startswith("M") else 1)
    (PROF / "ncu_traffic.json").write_text(json.dumps({
        "config": "C1", "kernel": "k_step_observe<1,1>",
        "source": f"profiles/{tag}_ncu_full.csv (ncu --set full, launch 5 of bench.py --steps 12)",
        "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "dram_bytes_per_launch": int(rd + wr)}) + "\n")
    md = [f"# {tag}: bench + ncu summary (B200, config C1)", "",
          f"bench: value {line['value']:.4g} {line['unit']}, {line['ms_per_step']:.4f} ms/step, fused kernel "
          f"{line['roofline']['kernel_ms'] * 1e3:.1f} us, roofline frac {line['roofline']['frac']:.3f}, "
          f"e2e {line.get('e2e', {}).get('value', float('nan')):.3g}", "",
          "| kernel | launches | mean (us, ncu serialised) | share |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        md.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot * 100:.1f}% |")
    md += ["", "| metric (k_step_observe, ncu --set full) | value |", "|---|---|"]
    for key, name in KEYS:
        if key in raw:
            md.append(f"| {name} | {raw[key][0]} {raw[key][1]} |")
    (PROF / f"{tag}_summary.md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1])
