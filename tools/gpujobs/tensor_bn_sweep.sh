for bn in 128 256; do
KP_F16TC_BN=$bn timeout 300 python tools/tensor_solve.py > /dev/null 2>&1 && KP_F16TC_BN=$bn timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_f16tc" --csv --log-file gpurun_out/tcbn_$bn.csv python tools/tensor_solve.py > /dev/null 2>&1
python - << PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/tcbn_$bn.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
v=[float(r[vi].replace(',','')) for r in rows[1:]]
print('BN=$bn n', len(v), 'per-position means (us):', [round(sum(v[i::4])/len(v[i::4])/1e3,1) for i in range(4)])
PY
done
KP_F16TC_BN=256 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tensor" 2>&1 | tail -1
