"""Split an ncu --set full capture of the trajectory kernel by code region
(instructions executed and stall samples), using the cubin's inline line
tables: every SASS instruction is charged to the innermost sim_kernel.cuh
frame of its inline chain.

    python tools/ncu_regions.py REPORT.ncu-rep BUILD/sim_inst_nw2.o MANGLED_SUBSTR [NTRAJ] [KERNEL_SUB]
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.environ.get('SABER_REGIONS_SRC', os.path.join(ROOT, 'paper_2506_19677_b200', 'csrc', 'sim_kernel.cuh'))
MARKS = [  # (region, first line containing the marker)
    ("gate_streak_g", "__device__ __forceinline__ void gate_streak_decisions("),
    ("gate_streak", "__device__ __forceinline__ void gate_streak_warp("),
    ("ledger_max", "// max over the ledger"),
    ("prologue", "// Simulates trajectory"),
    ("arrivals", "    // Arrivals due at t"),
    ("refresh", "      const int hc = hn;"),
    ("gate", "      } else if (!kWide && hn > 0) {"),
    ("gate_wide", "      if (kWide && hn > 0) {"),
    ("lowtier/static", "      } else if (low_head < low_tail) {"),
    ("streak_setup", "    if (t >= horizon) break;"),
    ("engine_quiet", "    const double nt = (horizon < t + tick)"),
    ("exact_pass", "      // Exact pass.  First make"),
    ("completion", "      if (ndone == 1) {"),
    ("end", "  if (failed && leader)"),
    ("kernel", "__global__ void __launch_bounds__"),
    ("streak_chunks", "__device__ __forceinline__ double streak_chunks("),
]


def regions():
    src = open(SRC).read().splitlines()
    starts = []
    for name, mark in MARKS:
        ln = [i + 1 for i, l in enumerate(src) if mark in l]
        if ln:
            starts.append((ln[0], name))
    starts.sort()
    return starts


def classify(chain, starts):
    for f, ln in chain:
        if f == "sim_kernel.cuh":
            name = "header"
            for a, n in starts:
                if ln >= a:
                    name = n
            return name
    return "other:" + (chain[0][0] if chain else "?")


def main():
    rep, obj, func_sub = sys.argv[1], sys.argv[2], sys.argv[3]
    ntraj = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    ksub = sys.argv[5] if len(sys.argv) > 5 else ""
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
    dis = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
    starts = regions()
    addr = {}
    func, pend, cur = None, [], []
    for l in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            func = m.group(1)
            continue
        m = re.search(r'//## File "(.*?)", line (\d+)', l)
        if m:
            pend.append((m.group(1).split("/")[-1], int(m.group(2))))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m:
            if pend:
                cur, pend = pend, []
            if func and func_sub in func:
                addr[int(m.group(1), 16)] = classify(cur, starts)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    heads = [i for i, x in enumerate(r) if x and x[0] == "Kernel Name"] + [len(r)]
    for a, b in zip(heads, heads[1:]):
        if ksub in r[a][1]:
            h, rows = r[a + 1], r[a + 2:b]
            break
    I = h.index
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
    base = None
    ts = ti = 0.0
    for x in rows:
        a = int(x[I("Address")], 16)
        base = a if base is None else base
        c = addr.get(a - base, "?")
        s = float(x[I("Warp Stall Sampling (All Samples)")] or 0)
        n = float(x[I("Instructions Executed")] or 0)
        agg[c][0] += s
        agg[c][1] += n
        agg[c][2] += 1
        ts += s
        ti += n
    print(f"{'region':16s} {'stall%':>7s} {'inst%':>7s} {'inst/traj':>10s} {'sass':>6s}")
    for k, (s, n, z) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:16s} {100 * s / ts:7.1f} {100 * n / ti:7.1f} {n / ntraj:10.0f} {z:6d}")
    print(f"{'total':16s} {'':7s} {'':7s} {ti / ntraj:10.0f} {sum(v[2] for v in agg.values()):6d}")


if __name__ == "__main__":
    main()
