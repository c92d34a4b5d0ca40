"""Aggregate an ncu SASS-page CSV by CUDA source line using nvdisasm line info."""
import csv, re, subprocess, sys, collections
rep, cubin, func_pat = sys.argv[1], sys.argv[2], sys.argv[3]
import os
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
# one section per profiled kernel: ["Kernel Name", name], header, rows...; pick by NCU_KERNEL_SUB
sub = os.environ.get("NCU_KERNEL_SUB", "")
starts = [i for i, x in enumerate(r) if x and x[0] == "Kernel Name"] + [len(r)]
for a, b in zip(starts, starts[1:]):
    if sub in r[a][1]:
        h = r[a + 1]; rows = r[a + 2:b]
        break
I = lambda n: h.index(n)
# nvdisasm with line info
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
func = None; line = None; addr2line = {}; lines = {}
for l in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m: func = m.group(1); continue
    m = re.search(r"//## File \"(.*?)\", line (\d+)", l)
    if m: line = (m.group(1).split("/")[-1], int(m.group(2))); continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and func and re.search(func_pat, func):
        addr2line[int(m.group(1), 16)] = line
base = None
agg = collections.defaultdict(lambda: [0.0, 0.0])
tot_i = tot_s = 0.0
for x in rows:
    a = int(x[I("Address")], 16)
    if base is None: base = a
    off = a - base
    ln = addr2line.get(off, ("?", 0))
    s = float(x[I("Warp Stall Sampling (All Samples)")] or 0); n = float(x[I("Instructions Executed")] or 0)
    agg[ln][0] += s; agg[ln][1] += n; tot_s += s; tot_i += n
src = {}
for ln in agg:
    if ln[0] != "?":
        try: src[ln] = open("/root/repo/paper_2506_19677_b200/csrc/" + ln[0]).read().splitlines()[ln[1]-1].strip()
        except Exception: src[ln] = ""
for ln, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{ln[0]}:{ln[1]:<5} stall {100*s/tot_s:5.1f}%  inst {100*n/tot_i:5.1f}%  {src.get(ln,'')[:90]}")
