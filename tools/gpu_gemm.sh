#!/bin/bash
# Per-launch merge GEMM table at cfg3: useful / padded flops (HPSB_TRACE) joined with ncu launch times.
cd "$GRAFT_REPO_ROOT"
HPSB_TRACE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:zgemm_grouped --csv \
  --log-file gpurun_out/gemm_launches.csv python tools/setup_probe.py 3 1 > gpurun_out/gemm_ncu.log 2> gpurun_out/gemm_trace.log
python - <<'PY' | tee gpurun_out/gemm_table.txt
import csv, re
rows = list(csv.reader(open('gpurun_out/gemm_launches.csv', errors='replace')))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[h]; vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
sc = {'ns': 1e-3, 'us': 1.0, 'ms': 1e3}
us = [float(r[vi].replace(',', '')) * sc.get(r[ui], 1.0) for r in rows[h + 1:] if len(r) > vi and r[vi]]
tr = [re.findall(r'descs (\d+) tiles (\d+) useful ([\d.e+]+) padded ([\d.e+]+)', l) for l in open('gpurun_out/gemm_trace.log')]
tr = [t[0] for t in tr if t]
print(len(us), len(tr))
tot = 0
print('launch descs tiles useful_GF padded_GF us useful_TF/s padded_TF/s')
for i, (u, t) in enumerate(zip(us, tr)):
    uf, pf = float(t[2]), float(t[3]); tot += u
    print(i, t[0], t[1], round(uf / 1e9, 2), round(pf / 1e9, 2), round(u, 1), round(uf / u / 1e6, 2), round(pf / u / 1e6, 2))
print('total us', tot)
PY
