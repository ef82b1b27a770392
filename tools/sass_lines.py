"""Attribute an ncu SASS source-page capture to CUDA source lines.
usage: python tools/sass_lines.py <ncu-rep> <cubin> <kernel-substring> [n]
Needs `nvdisasm -g` line info (build with -lineinfo).  Prints the source
lines with the most executed thread-instructions and stall samples."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
# line map for the kernel's .text section
line_of = {}
in_fn, cur = False, None
for ln in dis.splitlines():
    if ln.startswith(".text.") and kname in ln:
        in_fn = True
        continue
    if in_fn and ln.startswith(".text."):
        break
    if not in_fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m:
        line_of[int(m.group(1), 16)] = (cur, m.group(2).strip())
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kcur, hdr, data = None, None, collections.defaultdict(list)
for x in rows:
    if x and x[0] == "Kernel Name":
        kcur = x[1]
        continue
    if x and x[0] == "Address":
        hdr = x
        continue
    if kcur and hdr and len(x) > 5:
        data[kcur].append(x)
nk = sys.argv[5] if len(sys.argv) > 5 else "traj_kernel"
k = [k for k in data if nk in k][0]
v = data[k]
base = int(v[0][0], 16)
si, ti = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Thread Instructions Executed")
agg_t, agg_s = collections.Counter(), collections.Counter()
for x in v:
    off = int(x[0], 16) - base
    src = line_of.get(off, (("?", 0), ""))[0]
    agg_t[src] += float(x[ti] or 0)
    agg_s[src] += float(x[si] or 0)
T, S = sum(agg_t.values()), sum(agg_s.values())
src_lines = {}
for f in {s[0] for s in agg_t if s}:
    try:
        src_lines[f] = open(f"paper_2506_23364_b200/csrc/{f}").read().splitlines()
    except OSError:
        pass
print(f"{'file:line':22s} {'thr-inst%':>9s} {'stall%':>7s}  source")
for src, t in sorted(agg_t.items(), key=lambda kv: -kv[1])[:top]:
    f, n = src if src else ("?", 0)
    text = src_lines.get(f, [""] * (n + 1))[n - 1].strip() if f in src_lines and n else ""
    print(f"{f}:{n:<12d} {t / T * 100:9.2f} {agg_s[src] / S * 100:7.2f}  {text[:80]}")

# per-line opcode breakdown for the hottest lines (set OPS=1)
import os
if os.environ.get("OPS"):
    per = collections.defaultdict(collections.Counter)
    ii = hdr.index("Instructions Executed")
    for x in v:
        off = int(x[0], 16) - base
        src = line_of.get(off, (("?", 0), ""))[0]
        toks = x[1].split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
        per[src][op.split(".")[0]] += float(x[ii] or 0)
    W = sum(sum(c.values()) for c in per.values())
    for src, t in sorted(agg_t.items(), key=lambda kv: -kv[1])[:top]:
        c = per[src]
        print(f"{src[0]}:{src[1]}", ", ".join(f"{o} {n / W * 100:.2f}" for o, n in c.most_common(6)))
