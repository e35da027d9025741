mkdir -p gpurun_out/r02n
exec > gpurun_out/r02n/log.txt 2>&1
python tools/c4_batch_once.py 60 > gpurun_out/r02n/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none -k regex:gemm_f16x_kernel -s 4 -c 1 -o gpurun_out/r02n/early python tools/c4_batch_once.py 60 > gpurun_out/r02n/ncu1.log 2>&1; echo "early rc=$?"
timeout 1500 ncu --set full --clock-control none -k regex:gemm_f16x_kernel -s 200 -c 1 -o gpurun_out/r02n/late python tools/c4_batch_once.py 60 > gpurun_out/r02n/ncu2.log 2>&1; echo "late rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_f16x_kernel --csv --log-file gpurun_out/r02n/list.csv python tools/c4_batch_once.py 60 > gpurun_out/r02n/ncu3.log 2>&1; echo "list rc=$?"
python - << 'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r02n/list.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
v=[float(r[vi].replace(',',''))/1e3 for r in rows[1:]]
print('launches', len(v)); print('first 12 (us):', [round(x) for x in v[:12]]); print('by position in M-solve, iterations 1-3 vs 40-60:')
for p in range(4):
    a=v[4+p:16:4]; b=v[160+p:244:4]
    print(p, round(sum(a)/len(a)), round(sum(b)/len(b)))
PY
