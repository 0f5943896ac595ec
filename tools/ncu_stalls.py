"""Warp-stall samples of one kernel launch in an ncu report, aggregated by source line.

    python tools/ncu_stalls.py <report.ncu-rep> <kernel-id regex> <symbol substring> [cubin] [top]

kernel-id regex: ncu's ::regex:<name>:<invocation> selector (e.g. 'conv_pair_kernel:2');
symbol substring: a piece of the mangled name that identifies the instantiation in the local
cubin (e.g. 'conv_pair_kernelILi128E'); cubin: built with -lineinfo from the same sources
(default: compiles nothing, expects /tmp/<csrc file>.cubin).  SASS offsets are mapped to
source lines with nvdisasm -gi over the function's own .text section."""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rep, kid, sym = sys.argv[1], sys.argv[2], sys.argv[3]
cubin = sys.argv[4] if len(sys.argv) > 4 else None
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-id",
                      f"::regex:{kid}"], capture_output=True, text=True).stdout.splitlines()
ks = [i for i, l in enumerate(out) if l.startswith('"Kernel Name"')]
out = out[:ks[1]] if len(ks) > 1 else out
st = next(i for i, l in enumerate(out) if l.startswith('"Address"'))
rows = list(csv.reader(out[st:]))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
col = "Warp Stall Sampling (All Samples)"
base = int(rows[1][0], 16)

off2line = {}
if cubin:
    dis = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout.splitlines()
    in_fn, cur = False, "?"
    for ln in dis:
        m = re.match(r'\s*\.text\.(\S+):', ln)
        if m:
            in_fn = sym in m.group(1)
            continue
        if not in_fn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
        if m:
            f, l, f2, l2 = m.groups()
            cur = (f2 or f).split('/')[-1] + ':' + (l2 or l)
            continue
        m = re.match(r'\s+/\*([0-9a-f]{4,5})\*/\s+(\S.*)', ln)
        if m and not m.group(2).startswith('.'):
            off2line[int(m.group(1), 16)] = cur

agg = defaultdict(lambda: [0, defaultdict(int)])
tot = 0
for r in rows[1:]:
    s = int(r[ix[col]] or 0)
    tot += s
    k = off2line.get(int(r[0], 16) - base, r[1].strip()[:40])
    agg[k][0] += s
    for h in hdr:
        if h.startswith("stall_") and "Not Issued" not in h:
            agg[k][1][h] += int(r[ix[h]] or 0)
print(f"total samples {tot}")
for k, (v, rs) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    r2 = sorted(rs.items(), key=lambda x: -x[1])[:2]
    print(f"{v:7d} {100 * v / max(tot, 1):5.1f}%  {k:28s} {r2}")
