mkdir -p gpurun_out/r02i
exec > gpurun_out/r02i/log.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_batch.py -m gpu -q -x -k "band or operator or kronsum or batch or fused or solver" 2>&1 | tail -5; echo "tests rc=$?"
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "c1 or c4" 2>&1 | tail -3
for f in 1 0; do
  echo "KP_BAND_FUSED=$f"
  KP_BAND_FUSED=$f timeout 900 python bench.py --config C4 --no-tensor --no-cpu-baseline > gpurun_out/r02i/c4_$f.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r02i/c4_$f.json')); print('C4', d['value'])"
  KP_BAND_FUSED=$f timeout 900 python bench.py --config C1 --no-tensor --no-cpu-baseline --no-other-runs > gpurun_out/r02i/c1_$f.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r02i/c1_$f.json')); print('C1', d['value'], d['roofline_other']['kernel'], d['roofline_other']['frac'])"
done
KP_BAND_FUSED=1 timeout 600 python tools/c4_batch_profile.py 2>&1 | tail -8
