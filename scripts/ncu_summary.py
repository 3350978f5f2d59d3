"""Summarise ncu reports (gpurun_out/prof_<cfg>_<tag>.ncu-rep) into
profiles/ncu_<tag>.md and profiles/ncu_summary.json (bench.py reads the DRAM
traffic per launch of the dominant kernel from the latter)."""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = [
    ("gpu__time_duration.sum", "time_us"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_ld_conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem_st_conflicts"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "sm_ghz"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}


def report(path: Path):
    raw = path.with_suffix(".raw.csv")
    rawgz = path.with_suffix(".raw.csv.gz")
    if raw.exists():
        out = raw.read_text()
    elif rawgz.exists():
        import gzip

        out = gzip.open(rawgz, "rt").read()
    else:
        out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m, k in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if k in ("dram_read", "dram_write"):
                    v *= UNIT_SCALE.get(u, 1)
                if k == "time_us":
                    v *= UNIT_SCALE.get(u, 1) if u != "usecond" else 1
                d[k] = v
        res.append(d)
    return res


def main(tag):
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    summary_path = prof / "ncu_summary.json"
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {}
    lines = [f"# ncu summary ({tag})", "",
             "Captured with `ncu --set full --clock-control none` under gpurun (one B200), "
             "`scripts/round_r02.sh` / `scripts/prof_ncu.sh`; per-launch values (cold, serialised replays).", "",
             "| config | kernel | time us | DRAM read MB | DRAM write MB | DRAM % | L1/smem % | smem wavefronts | "
             "ld/st bank conflicts | tensor % | issue % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    g = ROOT / "gpurun_out"
    cfgs = sorted({q.name.split("_")[1] for q in list(g.glob(f"prof_*_{tag}.ncu-rep")) + list(g.glob(f"prof_*_{tag}.raw.csv"))
                   + list(g.glob(f"prof_*_{tag}.raw.csv.gz"))})
    for cfg in cfgs:
        rep = g / f"prof_{cfg}_{tag}.ncu-rep"
        ks = report(rep)
        for d in ks:
            short = d["kernel"].split("(")[0].replace("void ", "")
            lines.append(
                f"| {cfg} | `{short}` | {d.get('time_us', 0):.1f} | {d.get('dram_read', 0) / 1e6:.1f} | "
                f"{d.get('dram_write', 0) / 1e6:.1f} | {d.get('dram_pct', 0):.1f} | {d.get('l1tex_pct', 0):.1f} | "
                f"{d.get('smem_wavefronts', 0):.3g} | {d.get('smem_ld_conflicts', 0):.3g}/{d.get('smem_st_conflicts', 0):.3g} | "
                f"{d.get('tensor_pct', 0):.1f} | {d.get('issue_pct', 0):.1f} | {d.get('regs', 0):.0f} |")
        if ks:
            dom = max(ks, key=lambda d: d.get("time_us", 0))
            summary[cfg] = {"tag": tag, "kernel": dom["kernel"],
                            "dram_bytes_per_launch": dom.get("dram_read", 0) + dom.get("dram_write", 0),
                            "time_us": dom.get("time_us"), "launches": ks}
    (prof / f"ncu_{tag}.md").write_text("\n".join(lines) + "\n")
    summary_path.write_text(json.dumps(summary, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
