timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tensor" 2>&1 | tail -2
timeout 300 python tools/tensor_solve.py > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_f16tc" --csv --log-file gpurun_out/launches_tc1.csv python tools/tensor_solve.py > /dev/null 2>&1
python - << 'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_tc1.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
v=[float(r[vi].replace(',','')) for r in rows[1:]]
print('n', len(v), 'G1..G4 means (us):', [round(sum(v[i::4])/len(v[i::4])/1e3,1) for i in range(4)])
PY
timeout 900 python bench.py --no-dense --no-cpu-baseline > gpurun_out/bench_tc1.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_tc1.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['tensor_mode'])"
