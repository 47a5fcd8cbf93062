"""Summarise ncu launch lists of `profiles/prof_codec.py <eb> 26 <block_version>` (one warm-up
and one measured compress + decompress of the config-2 vector, n = 2^26, one bound per run;
metrics gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum, --clock-control
none) into profiles/ncu_summary.json, keyed by the bench's kernel groups.

    python profiles/make_ncu_summary.py profiles/ncu_summary.json 1e-3=a.csv 1e-4=b.csv 1e-6=c.csv [v1:1e-3=d.csv ...]

The measured round trip is the second one of each run (launches after the second
lc_range_kernel).  `bench.py` reads `dram_bytes_per_launch` of its dominant group as the
roofline's `traffic`."""
import collections
import csv
import json
import sys

GROUPS = {
    'range': ['lc_range_kernel', 'lc_quant_setup_kernel'],
    'quantizer': ['lc_anchor_tiles_kernel', 'lc_anchor_scan_kernel', 'lc_quant_wa_kernel', 'lc_map_scan_kernel',
                  'lc_quant_wfix_kernel', 'lc_sync_starts_kernel', 'lc_histw_kernel', 'lc_hist16_kernel', 'lc_hist_kernel',
                  'lc_quant_serial_kernel'],
    'encoder': ['lc_codebook_kernel', 'lc_zero_words_kernel', 'lc_encode_kernel'],
    'decode_v3': ['lc_dec_tables_kernel', 'lc_dec_v3_kernel'],
    'huffman_decode': ['lc_dec_tables_kernel', 'lc_dec_sync_kernel', 'lc_dec_fix_kernel', 'lc_dec_scan_kernel',
                       'lc_dec_write_kernel', 'lc_dec_status_kernel'],
    'reconstruction': ['lc_set_first_kernel', 'lc_rec_a_kernel', 'lc_map_scan_kernel', 'lc_rec_b_kernel',
                       'lc_rec_final_kernel', 'lc_rec_serial_kernel'],
}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'),
                          h.index('Metric Unit'), h.index('ID'))
    out = collections.OrderedDict()
    for r in rows[1:]:
        d = out.setdefault(r[ii], {'kernel': r[ki].split('(')[0].replace('void ', '').split('<')[0]})
        v = float(r[vi].replace(',', ''))
        u = r[ui]
        if r[mi].startswith('dram__bytes'):
            d['dram'] = d.get('dram', 0) + v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
        elif r[mi] == 'gpu__time_duration.sum':
            d['us'] = v / 1000 if u.startswith('n') else (v if u.startswith('u') else v * 1000)
    return list(out.values())


def measured(ls):
    starts = [i for i, d in enumerate(ls) if d['kernel'] == 'lc_range_kernel']
    return ls[starts[-1]:]


def split(ls):
    """compress = up to the last encoder kernel; decompress = the rest."""
    last_enc = max(i for i, d in enumerate(ls) if d['kernel'] == 'lc_encode_kernel')
    return ls[:last_enc + 1], ls[last_enc + 1:]


out = {'source': 'ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none '
                 'python profiles/prof_codec.py <eb> 26 <block_version>; second (measured) round trip; per-launch times '
                 'are cold-cache and serialised', 'runs': {}}
acc = collections.defaultdict(lambda: collections.defaultdict(list))
for arg in sys.argv[2:]:
    tag, path = arg.split('=', 1)
    fmt = 'v3'
    if ':' in tag:
        fmt, tag = tag.split(':', 1)
    comp, dec = split(measured(launches(path)))
    run = {}
    for g, ks in GROUPS.items():
        part = comp if g in ('range', 'quantizer', 'encoder') else dec
        if g == 'decode_v3' and not any(d['kernel'] == 'lc_dec_v3_kernel' for d in dec):
            continue
        if g in ('huffman_decode', 'reconstruction') and any(d['kernel'] == 'lc_dec_v3_kernel' for d in dec):
            continue
        if g == 'reconstruction':
            lo = [i for i, d in enumerate(part) if d['kernel'] in ('lc_set_first_kernel', 'lc_rec_a_kernel')]
            part = part[lo[0]:] if lo else []
        elif g == 'huffman_decode':
            hi = [i for i, d in enumerate(part) if d['kernel'] in ('lc_set_first_kernel', 'lc_rec_a_kernel')]
            part = part[:hi[0]] if hi else part
        sel = [d for d in part if d['kernel'] in ks]
        if not sel:
            continue
        run[g] = {'us': round(sum(d.get('us', 0) for d in sel), 1), 'dram_bytes': int(sum(d.get('dram', 0) for d in sel)),
                  'kernels': [(d['kernel'], round(d.get('us', 0), 1), int(d.get('dram', 0))) for d in sel]}
        acc[fmt + ':' + g]['us'].append(run[g]['us'])
        acc[fmt + ':' + g]['dram'].append(run[g]['dram_bytes'])
    run['compress_us'] = round(sum(d.get('us', 0) for d in comp), 1)
    run['decompress_us'] = round(sum(d.get('us', 0) for d in dec), 1)
    out['runs'][fmt + ':' + tag] = run
for key, d in acc.items():
    fmt, g = key.split(':', 1)
    ent = {'dram_bytes_per_launch': sum(d['dram']) / len(d['dram']), 'ncu_us_per_launch': sum(d['us']) / len(d['us']),
           'bounds': len(d['us'])}
    if fmt == 'v3' or g not in out:
        out[g] = ent
json.dump(out, open(sys.argv[1], 'w'), indent=1)
for k, v in out.items():
    if isinstance(v, dict) and 'dram_bytes_per_launch' in v:
        print(k, 'dram MB/launch %.1f' % (v['dram_bytes_per_launch'] / 1e6), 'ncu us %.0f' % v['ncu_us_per_launch'])
for tag, run in out['runs'].items():
    print(tag, 'compress', run['compress_us'], 'decompress', run['decompress_us'],
          {g: (r['us'], round(r['dram_bytes'] / 1e6)) for g, r in run.items() if isinstance(r, dict)})
