mkdir -p gpurun_out
for c in c2 c2_n32 c2_fused; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench7_$c.json 2> gpurun_out/bench7_$c.err; tail -2 gpurun_out/bench7_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench7_$c.json'))
print('$c', round(d['value']/1e9,2), 'Gval/s', round(d['ms_per_step'],2), 'ms', 'count', d['count'], 'GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2), d['launch'])
"
done
python bench.py --config c2_fused --steps 1 --warmup 1 > gpurun_out/plain_c2f.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2f.csv python bench.py --config c2_fused --steps 1 --warmup 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_c2f.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:]: print(r[ki][:50], r[vi])
PY
