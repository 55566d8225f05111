import csv, sys, subprocess, collections
def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None; out = []
    for r in rows:
        if 'Kernel Name' in r: hdr = r; continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get('Metric Name') == 'gpu__time_duration.sum':
                out.append((d['Kernel Name'], float(d['Metric Value'].replace(',','')), d['Metric Unit']))
    return out
def raw(path, names):
    txt = subprocess.run(['ncu','-i',path,'--page','raw','--csv'],capture_output=True,text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, u = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {n: (row[h.index(n)], u[h.index(n)]) for n in names if n in h}
        d['Kernel Name'] = row[h.index('Kernel Name')][:70]
        res.append(d)
    return res
if __name__ == '__main__':
    mode = sys.argv[1]
    if mode == 'launches':
        agg = collections.OrderedDict()
        for n, t, u in launches(sys.argv[2]):
            k = n[:80]
            agg.setdefault(k, []).append(t)
        tot = sum(sum(v) for v in agg.values())
        for k, v in agg.items():
            print(f"{k:80s} n={len(v):4d} mean={sum(v)/len(v):12.1f} share={sum(v)/tot*100:5.1f}% ({u})")
    else:
        names = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed','sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_elapsed','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','launch__registers_per_thread','sm__throughput.avg.pct_of_peak_sustained_elapsed','launch__grid_size','sm__warps_active.avg.pct_of_peak_sustained_active']
        extra = sys.argv[3:] 
        for d in raw(sys.argv[2], names + extra):
            print(d)
