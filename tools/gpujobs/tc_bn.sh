# tcgen05 tile width for the tensor-mode M-solve products: 192 vs 256 (and 128)
exec > gpurun_out/tcbn/log.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k tensor 2>&1 | tail -1
KP_F16TC_BN=192 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k tensor 2>&1 | tail -1
for bn in 256 192 128; do
  echo "bn=$bn"
  KP_F16TC_BN=$bn timeout 600 python bench.py --no-cpu-baseline --no-other-runs --no-dense 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['tensor_mode']; print(t['value'], t['roofline']['frac'], t['final_rel_err'])"
done
