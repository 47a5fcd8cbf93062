"""Instruction and stall-sample shares of source-line regions of one kernel.
    python profiles/ncu_regions.py report.ncu-rep <kernel regex> file:lo-hi=name ...  (plus n_elements)"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
specs = []
nel = None
for a in sys.argv[3:]:
    if '=' not in a:
        nel = float(eval(a))
        continue
    loc, name = a.split('=')
    f, rng = loc.split(':')
    lo, hi = (int(v) for v in rng.split('-'))
    specs.append((f, lo, hi, name))
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', 'regex:' + kern,
                      '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
rows = []
f = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == 'File Path':
        f = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        continue
    if hdr and r[0].isdigit() and r[2] == '-':
        rows.append((f, int(r[0]), int(r[7] or 0), int(r[4] or 0)))
ti = sum(x[2] for x in rows)
ts = sum(x[3] for x in rows)
reg = collections.Counter()
regs = collections.Counter()
for fi, ln, ins, smp in rows:
    name = 'other:' + fi
    for sf, lo, hi, nm in specs:
        if fi == sf and lo <= ln <= hi:
            name = nm
            break
    reg[name] += ins
    regs[name] += smp
for k, v in reg.most_common():
    extra = f"  {v * 32 / nel:6.1f} thread-instr/elem" if nel else ""
    print(f"{k:26s} ins {100 * v / ti:5.1f}%  samples {100 * regs[k] / ts:5.1f}%{extra}")
print('total warp instr', ti, (f"= {ti * 32 / nel:.1f} thread-instr/elem" if nel else ""))
