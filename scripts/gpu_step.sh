python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_predictor.py tests/test_gpu_masks.py -x -q 2>&1 | tail -3
for w in pred step; do timeout 120 python scripts/prof_attn.py $w 10; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_step.csv python scripts/prof_attn.py step 2 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/launches_step.csv')) if len(r)>5]
h=rows[0]; i=h.index('Kernel Name'); m=h.index('Metric Value')
agg=collections.OrderedDict()
for r in rows[1:]:
    if 'sv::' in r[i]: agg.setdefault(r[i][:50],[]).append(float(r[m]))
for k,v in agg.items(): print(len(v), '%.1f us' % (sum(v)/len(v)/1e3), k)
PY
