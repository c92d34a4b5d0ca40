import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
keep = ["Duration", "Elapsed Cycles", "SM Active Cycles", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Achieved Active Warps Per SM", "Registers Per Thread",
        "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Issued Instructions", "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput", "Theoretical Occupancy",
        "Dynamic Shared Memory Per Block", "Branch Efficiency", "Grid Size"]
for x in r[1:]:
    if x[h.index("Metric Name")] in keep:
        print(x[h.index("Metric Name")].ljust(40), x[h.index("Metric Value")], x[h.index("Metric Unit")])
