"""Summarise an ncu --set full capture of one kernel (run here, no GPU):
headline SOL / occupancy / issue metrics, FP64 pipe and DRAM bytes, opcode
mix and stall reasons from the SASS source page.
usage: python tools/ncu_summary.py gpurun_out/prof_traj.ncu-rep [kernel-substring]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kname = sys.argv[2] if len(sys.argv) > 2 else "traj_kernel"


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kname}", *args], capture_output=True, text=True).stdout


r = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = r[0]
mi, ui, vi = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
keep = ["Duration", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Grid Size", "Block Size"]
seen = set()
for row in r[1:]:
    if row[mi] in keep and row[mi] not in seen:
        seen.add(row[mi])
        print(f"{row[mi]:34s} {row[vi]:>18s} {row[ui]}")
rr = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
H, U, V = rr[0], rr[1], rr[2]
for name in ["dram__bytes_read.sum", "dram__bytes_write.sum",
             "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
             "TPC.TriageCompute.sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed",
             "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
             "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum"]:
    if name in H:
        i = H.index(name)
        print(f"{name.split('.')[-2] if 'TriageCompute' in name else name:34s} {V[i]:>18s} {U[i]}")

rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
cur, hdr, data = None, None, collections.defaultdict(list)
for x in rows:
    if x and x[0] == "Kernel Name":
        cur = x[1]
        continue
    if x and x[0] == "Address":
        hdr = x
        continue
    if cur and hdr and len(x) > 5:
        data[cur].append(x)
mains = [k for k in data if kname in k]
if mains:
    v = data[mains[0]]
    si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    ti = hdr.index("Thread Instructions Executed")
    stalls = [s for s in hdr if s.startswith("stall_") and "Not Issued" not in s]
    ops, st = collections.Counter(), collections.Counter()
    for x in v:
        toks = x[1].split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
        ops[op.split(".")[0]] += float(x[ii] or 0)
        for s in stalls:
            st[s] += float(x[hdr.index(s)] or 0)
    tot = sum(ops.values())
    thr = sum(float(x[ti] or 0) for x in v)
    print(f"\nwarp-instructions {tot:.4e}  thread-instructions {thr:.4e}")
    print("opcode mix (% of warp-instructions):", ", ".join(f"{o} {n / tot * 100:.1f}" for o, n in ops.most_common(16)))
    ts = sum(st.values())
    print("stall reasons (% of samples):", ", ".join(f"{s[6:]} {n / ts * 100:.1f}" for s, n in st.most_common(8)))
