# BN small-layer latency: fused cooperative vs two-launch; ncu kernel durations
mkdir -p gpurun_out
for s in 1024x4 1024x16 128x128; do
python tools/bench_bn.py --only $s --dtype f32 2>&1 | grep -v "^{" | sed "s/^/fused   /"
RP_BN_UNFUSED=1 python tools/bench_bn.py --only $s --dtype f32 2>&1 | grep -v "^{" | sed "s/^/unfused /"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bn_small_ncu.csv python tools/bench_bn.py --only 1024x4 --iters 3 > /dev/null 2>&1
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/bn_small_ncu.csv')))
h=None
for r in rows:
    if 'Kernel Name' in r: h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r))
        if d.get('Metric Name')=='gpu__time_duration.sum': print(d['Kernel Name'][:60], d['Metric Value'], d['Metric Unit'])
P
