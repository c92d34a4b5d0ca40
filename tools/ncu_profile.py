"""Summarise an `ncu --set full` capture of the engine's kernels into profiles/.

    python tools/ncu_profile.py REPORT.ncu-rep OUT.txt [--traffic-json OUT.json]
           [--label SUB=NAME:TRAJ ...] [--tag r02c] [--commit SHA] [--title TEXT]

OUT.txt gets, per kernel, the headline metrics (duration, issue-slot %, warps
active, threads per instruction, FP64 pipe %, DRAM bytes, registers) and the
top stall reasons in cycles per issued instruction.  --traffic-json writes the
machine-readable record bench.py reports beside its live FP64 roofline
(roofline.issue / roofline.traffic), stamped with the tag and the commit the
capture was taken at.  --label maps a kernel-name substring to a short name and
the trajectories that launch simulated (e.g. "0, 0, 2>=sim_kernel<SABER>:3840").
"""
import argparse
import csv
import json
import subprocess
import sys

HEAD = [("gpu__time_duration.sum", "duration"),
        ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots busy %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads per instruction (of 32)"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst %"),
        ("smsp__inst_executed.sum", "warp instructions"),
        ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("launch__registers_per_thread", "registers"),
        ("launch__grid_size", "grid"),
        ("sm__warps_active.avg.per_cycle_active", "warps per SM")]
STALL = "smsp__average_warps_issue_stalled_"


def scaled(v, unit):
    x = float(v.replace(",", ""))
    return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(unit, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--traffic-json")
    ap.add_argument("--label", action="append", default=[])
    ap.add_argument("--tag", default="")
    ap.add_argument("--commit", default="")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    col = {n: i for i, n in enumerate(h)}
    labels = []
    for spec in a.label:
        sub, rest = spec.split("=", 1)
        name, traj = rest.rsplit(":", 1)
        labels.append((sub, name, int(traj)))
    lines = [f"# {a.title or 'ncu --set full --clock-control none'}"
             f"{' — ' + a.tag if a.tag else ''}{' @ ' + a.commit if a.commit else ''}", ""]
    kernels = {}
    dram_total = 0.0
    for r in data:
        kname = r[col["Kernel Name"]]
        short = kname
        traj = None
        for sub, name, t in labels:
            if sub in kname:
                short, traj = name, t
        lines.append(f"## {short}   ({kname})")
        rec = {}
        for m, title in HEAD:
            if m not in col:
                continue
            v, u = r[col[m]], units[col[m]]
            lines.append(f"   {title:<34} {v} {u}")
            rec[m] = v
        rd = scaled(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
        wr = scaled(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
        dram_total += rd + wr
        stalls = []
        for n, i in col.items():
            if n.startswith(STALL) and n.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), n[len(STALL):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        lines.append("   stall reasons (cycles per issued instruction):")
        for v, n in stalls[:8]:
            lines.append(f"      {n:<24} {v:.3f}")
        lines.append("")
        dur_ms = float(r[col["gpu__time_duration.sum"]]) * (1e-3 if units[col["gpu__time_duration.sum"]] == "us" else 1.0)
        kernels[short] = {
            "trajectories": traj,
            "duration_ms_under_ncu": dur_ms,
            "issue_active_pct": float(rec["sm__inst_issued.avg.pct_of_peak_sustained_active"]),
            "warps_active_pct": float(rec["sm__warps_active.avg.pct_of_peak_sustained_active"]),
            "fp64_pipe_active_pct": float(rec["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
            "threads_per_inst": float(rec["smsp__thread_inst_executed_per_inst_executed.ratio"]),
            "registers": int(float(rec["launch__registers_per_thread"])),
            "warp_instructions": float(rec["smsp__inst_executed.sum"].replace(",", "")),
            "dram_bytes": rd + wr,
            "top_stalls": {n: v for v, n in stalls[:4]},
        }
    tot = sum(k["duration_ms_under_ncu"] for k in kernels.values())
    weighted = sum(k["issue_active_pct"] * k["duration_ms_under_ncu"] for k in kernels.values()) / tot
    lines.append(f"issue slots busy, time-weighted over these kernels: {weighted:.1f} %")
    lines.append(f"DRAM bytes, all kernels: {dram_total / 1e6:.2f} MB")
    open(a.out, "w").write("\n".join(lines) + "\n")
    if a.traffic_json:
        json.dump({"source": f"tools/ncu_profile.py {a.report} ({a.title})", "tag": a.tag,
                   "commit": a.commit, "dram_bytes_per_launch": dram_total, "kernels": kernels,
                   "issue_active_pct_weighted": weighted}, open(a.traffic_json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
