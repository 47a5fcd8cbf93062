"""One-screen summary of a kernel in an ncu --set full report (duration, throughput,
issue activity, occupancy, DRAM bytes).  python profiles/ncu_brief.py report.ncu-rep [kernel regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = ['ncu', '-i', rep, '--page', 'details', '--csv']
if len(sys.argv) > 2:
    args += ['--kernel-name', 'regex:' + sys.argv[2]]
out = subprocess.run(args, capture_output=True, text=True).stdout
want = ('Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Issue Slots Busy',
        'Executed Ipc Active', 'Achieved Occupancy', 'Registers Per Thread', 'No Eligible',
        'Eligible Warps Per Scheduler', 'L2 Hit Rate', 'Warp Cycles Per Issued Instruction', 'Grid Size')
r = list(csv.reader(io.StringIO(out)))
h = r[0]
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get('Metric Name') in want:
        print(f"{d['Kernel Name'][:28]:28s} {d['Metric Name']:36s} {d['Metric Value']:>12s} {d['Metric Unit']}")
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'] + args[5:], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    hh = rr[0]
    for row in rr[2:]:
        d = dict(zip(hh, row))
        rd = float(d.get('dram__bytes_read.sum', 'nan').replace(',', '') or 'nan')
        wr = float(d.get('dram__bytes_write.sum', 'nan').replace(',', '') or 'nan')
        print(f"{d.get('Kernel Name', '')[:28]:28s} dram read {rd} {rr[1][hh.index('dram__bytes_read.sum')]} write {wr}")
