mkdir -p gpurun_out
AB_ROUNDS=2 timeout 2400 python tools/ab_fwd.py "" f2fp f2fpp1 f2fpp2 p1 > gpurun_out/r02f_ab.txt 2>&1
python - <<'PY'
import json, collections
rows=[json.loads(l) for l in open('gpurun_out/r02f_ab.txt') if l.startswith('{')]
agg=collections.defaultdict(list)
for r in rows:
    if 'tflops' in r: agg[(tuple(r['shape']), r['variant'])].append((r['tflops'], r['sm_mhz']))
for k,v in sorted(agg.items()): print(k, [f"{t:.0f}@{m:.0f}" for t,m in v])
PY
