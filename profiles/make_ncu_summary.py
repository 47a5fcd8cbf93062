"""Summarise an ncu metrics CSV (dram bytes + duration per launch) into
profiles/ncu_summary.json keyed by the bench's kernel groups."""
import csv, json, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit'), h.index('ID')
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
seq = list(launch.values())
# split into the 6 iterations (2 per bound) at lc_anchor_tiles_kernel; keep the second of each bound
its, cur = [], None
for d in seq:
    if d['kernel'] == 'lc_anchor_tiles_kernel':
        cur = []; its.append(cur)
    cur.append(d)
groups = {'quantizer': ['lc_quant_a_kernel', 'lc_map_scan_kernel', 'lc_quant_b_kernel'],
          'encoder': ['lc_codebook_kernel', 'lc_zero_words_kernel', 'lc_encode_kernel'],
          'huffman_decode': ['lc_dec_tables_kernel', 'lc_dec_sync_kernel', 'lc_dec_fix_kernel', 'lc_dec_scan_kernel',
                             'lc_dec_write_kernel', 'lc_dec_status_kernel'],
          'reconstruction': ['lc_rec0_kernel', 'lc_rec0_scan_kernel', 'lc_rec_a_kernel', 'lc_map_scan_kernel', 'lc_rec_b_kernel']}
out = {}
bounds = ['1e-3', '1e-4', '1e-6']
for g, ks in groups.items():
    per = {}
    for bi, it in enumerate(its[1::2]):
        # reconstruction's map_scan is the second one in the iteration
        if g == 'reconstruction':
            idx = [i for i, d in enumerate(it) if d['kernel'] == 'lc_rec0_kernel'][0]
            sel = [d for d in it[idx:] if d['kernel'] in ks]
        elif g == 'quantizer':
            idx = [i for i, d in enumerate(it) if d['kernel'] == 'lc_quant_a_kernel'][0]
            sel = [d for d in it[idx:idx + 3] if d['kernel'] in ks]
        else:
            sel = [d for d in it if d['kernel'] in ks]
        per[bounds[bi]] = {'dram_bytes': sum(d.get('dram', 0) for d in sel), 'us': sum(d.get('us', 0) for d in sel),
                           'kernels': [(d['kernel'], round(d.get('us', 0), 1), int(d.get('dram', 0))) for d in sel]}
    out[g] = {'dram_bytes_per_launch': sum(p['dram_bytes'] for p in per.values()) / len(per),
              'ncu_us_per_launch': sum(p['us'] for p in per.values()) / len(per), 'per_bound': per,
              'source': 'ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum '
                        '--clock-control none, scratch/prof_pipe.py 1e-3 1e-4 1e-6 (n=2^26), second call per bound'}
json.dump(out, open(sys.argv[2], 'w'), indent=1)
for g, d in out.items():
    print(g, 'dram MB/launch %.1f' % (d['dram_bytes_per_launch'] / 1e6), 'ncu us %.0f' % d['ncu_us_per_launch'])
