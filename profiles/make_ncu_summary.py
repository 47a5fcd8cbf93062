"""Summarise an ncu launch list of `bench.py --steps 1 --warmup 1 --no-cpu --no-solver`
(metrics gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum) into
profiles/ncu_summary.json keyed by the bench's kernel groups.

    python profiles/make_ncu_summary.py launches.csv profiles/ncu_summary.json

Every compress+decompress round trip starts with lc_range_kernel; the second
step's three round trips (bounds 1e-3, 1e-4, 1e-6) are summarised."""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui, ii = (h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'),
                      h.index('Metric Unit'), h.index('ID'))
launch = collections.OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[ii], {'kernel': r[ki].split('(')[0].replace('void ', '').split('<')[0]})
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    if r[mi].startswith('dram__bytes'):
        v *= {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
        d['dram'] = d.get('dram', 0) + v
    elif r[mi] == 'gpu__time_duration.sum':
        d['us'] = v / 1000 if u in ('ns', 'nsecond') else (v if u in ('us', 'usecond') else v * 1000)
its, cur = [], None
for d in launch.values():
    if d['kernel'] == 'lc_range_kernel':
        cur = []
        its.append(cur)
    if cur is not None:
        cur.append(d)
timed = its[3:6]
groups = {'quantizer': ['lc_anchor_tiles_kernel', 'lc_anchor_scan_kernel', 'lc_quant_a_kernel', 'lc_map_scan_kernel',
                        'lc_quant_b_kernel', 'lc_hist16_kernel'],
          'encoder': ['lc_codebook_kernel', 'lc_zero_words_kernel', 'lc_encode_kernel'],
          'huffman_decode': ['lc_dec_tables_kernel', 'lc_dec_sync_kernel', 'lc_dec_fix_kernel', 'lc_dec_scan_kernel',
                             'lc_dec_write_kernel', 'lc_dec_status_kernel'],
          'reconstruction': ['lc_rec_a_kernel', 'lc_map_scan_kernel', 'lc_rec_b_kernel', 'lc_rec_final_kernel']}
out = {}
bounds = ['1e-3', '1e-4', '1e-6']
for g, ks in groups.items():
    per = {}
    for bi, it in enumerate(timed):
        names = [d['kernel'] for d in it]
        if g == 'reconstruction':
            lo = names.index('lc_rec_a_kernel')
            sel = [d for d in it[lo:] if d['kernel'] in ks]
        elif g == 'quantizer':
            hi = names.index('lc_quant_b_kernel') + 1
            if hi < len(names) and names[hi] == 'lc_hist16_kernel':
                hi += 1
            sel = [d for d in it[:hi] if d['kernel'] in ks]
        else:
            sel = [d for d in it if d['kernel'] in ks]
        per[bounds[bi]] = {'dram_bytes': sum(d.get('dram', 0) for d in sel), 'us': sum(d.get('us', 0) for d in sel),
                           'kernels': [(d['kernel'], round(d.get('us', 0), 1), int(d.get('dram', 0))) for d in sel]}
    out[g] = {'dram_bytes_per_launch': sum(p['dram_bytes'] for p in per.values()) / len(per),
              'ncu_us_per_launch': sum(p['us'] for p in per.values()) / len(per), 'per_bound': per,
              'source': 'ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum '
                        '--clock-control none, bench.py --steps 1 --warmup 1 --no-cpu --no-solver (n=2^26), '
                        'timed step'}
other = collections.defaultdict(float)
for it in timed:
    for d in it:
        if d['kernel'] == 'lc_range_kernel' or d['kernel'] == 'lc_range_final_kernel':
            other[d['kernel']] += d.get('us', 0) / 3
out['range'] = {'ncu_us_per_launch': sum(other.values()), 'kernels': dict(other)}
json.dump(out, open(sys.argv[2], 'w'), indent=1)
for g, d in out.items():
    print(g, 'dram MB/launch %.1f' % (d.get('dram_bytes_per_launch', 0) / 1e6), 'ncu us %.0f' % d['ncu_us_per_launch'])
