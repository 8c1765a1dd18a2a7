"""Print per-launch metrics from an ncu --csv launch list."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = collections.OrderedDict()
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        out.setdefault((int(d['ID']), d['Kernel Name'][:60]), {})[d['Metric Name']] = d['Metric Value']
for (i, n), m in out.items():
    g = lambda k: float(m.get(k, 'nan').replace(',', ''))
    print(f"{i:>4} {n:60s} t={g('gpu__time_duration.sum')/1000:7.2f}us rd={g('dram__bytes_read.sum')/1e6:6.2f}MB "
          f"wr={g('dram__bytes_write.sum')/1e6:6.2f}MB warps={m.get('sm__warps_active.avg.pct_of_peak_sustained_active','')} "
          f"grid={m.get('launch__grid_size','')}")
