"""Summarise bench JSON lines and ncu launch CSVs from gpurun_out (dev tool)."""
import csv, glob, json, sys
tag = sys.argv[1]
for f in sorted(glob.glob(f'/root/repo/gpurun_out/{tag}_*.json')):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
        r = j.get('roofline', {})
        print(f.split('/')[-1], round(j['value'] / 1e6, 3), 'M/s', round(j['ms_per_step'] * 1e3, 1), 'us',
              'kern', round(r.get('kernel_us', 0), 1), 'launches', j.get('gpu_launches'))
    except Exception as e:
        print(f.split('/')[-1], 'ERR', e)
for f in sorted(glob.glob(f'/root/repo/gpurun_out/{tag}_ncu*.csv')):
    rows = [ln for ln in open(f) if ln.startswith('"')]
    agg = {}
    for x in csv.DictReader(rows):
        k = (x['Kernel Name'].split('<')[0].replace('void ', ''), x['Metric Name'])
        agg.setdefault(k, []).append(float(x['Metric Value'].replace(',', '')))
    print(f.split('/')[-1])
    for (kn, m), v in sorted(agg.items()):
        print('   ', kn, m, round(sum(v) / len(v) / (1e3 if 'time' in m else 1e6), 2), 'us' if 'time' in m else 'MB', 'n', len(v))
