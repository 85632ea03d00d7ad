"""Development aid: per-CUDA-source-line warp-stall samples and executed
instructions of one kernel, joining ncu's SASS source page (csv) with the
line table of the built cubin (nvdisasm -g).

    python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX MANGLED_SUBSTR [top]
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, kre, fsub = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
obj = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1606_06659_b200/lib/sweep_kernels.o")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                      text=True).stdout.split("\n")
cur, line, off2line = None, None, {}
for l in sass:
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        cur = m.group(1)
        continue
    if cur is None or fsub not in cur:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and line:
        off2line[int(m.group(1), 16)] = line
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kre}", "--launch-count", "1"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
hdr, data = rows[hi], rows[hi + 1:]
si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
seen, base = set(), None
samp, inst = collections.Counter(), collections.Counter()
for d in data:
    if not d[0].startswith("0x") or d[0] in seen:
        continue
    seen.add(d[0])
    a = int(d[0], 16)
    base = a if base is None else min(base, a)
for d in data:
    if not d[0].startswith("0x"):
        continue
    key = (d[0], d[1])
    if key in seen and isinstance(seen, set) and False:
        continue
tot_s = tot_i = 0
done = set()
for d in data:
    if not d[0].startswith("0x") or d[0] in done:
        continue
    done.add(d[0])
    ln = off2line.get(int(d[0], 16) - base, ("?", 0))
    s = int(d[si] or 0)
    i = int(d[ie] or 0)
    samp[ln] += s
    inst[ln] += i
    tot_s += s
    tot_i += i
src = {}
for f in set(k[0] for k in samp):
    p = os.path.join(os.path.dirname(obj), "..", "csrc", f)
    if os.path.exists(p):
        src[f] = open(p).read().split("\n")
print(f"total samples {tot_s}, warp instructions {tot_i}")
for ln, s in samp.most_common(top):
    text = src.get(ln[0], [])[ln[1] - 1].strip() if ln[0] in src and ln[1] else ""
    print(f"{s / tot_s * 100:5.1f}% smp {inst[ln] / tot_i * 100:5.1f}% inst  {ln[0]}:{ln[1]:<5} {text[:90]}")
