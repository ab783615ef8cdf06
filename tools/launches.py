"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections, csv, sys

def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    recs = collections.OrderedDict()
    for r in rows:
        if r and r[0] == 'ID':
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = d['ID']
            rec = recs.setdefault(key, {'name': d['Kernel Name'], 'grid': d['Grid Size']})
            v = float(d['Metric Value'].replace(',', ''))
            unit = d['Metric Unit']
            scale = {'ns': 1, 'us': 1e3, 'ms': 1e6, 'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(unit, 1)
            rec[d['Metric Name']] = v * scale
    return list(recs.values())

if __name__ == '__main__':
    recs = load(sys.argv[1])
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for r in recs:
        name = r['name'].split('(')[0][:48]
        t = tot[name]
        t[0] += 1
        t[1] += r.get('gpu__time_duration.sum', 0)
        t[2] += r.get('dram__bytes_read.sum', 0)
        t[3] += r.get('dram__bytes_write.sum', 0)
    T = sum(v[1] for v in tot.values())
    for name, v in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"{name:48s} n={v[0]:3d} {v[1]/1e6:8.3f} ms ({100*v[1]/T:5.1f}%)  rd {v[2]/1e9:7.2f} GB  wr {v[3]/1e9:7.2f} GB  {(v[2]+v[3])/max(v[1],1):6.0f} GB/s")
    print(f"total {T/1e6:.3f} ms over {len(recs)} launches")
    if len(sys.argv) > 2:
        for r in recs:
            print(r['name'].split('(')[0][:40], r['grid'], '%.1f us' % (r.get('gpu__time_duration.sum', 0) / 1e3),
                  '%.2f GB' % ((r.get('dram__bytes_read.sum', 0) + r.get('dram__bytes_write.sum', 0)) / 1e9))
