# C4 throughput: fp16 tile width and stream count variants
exec > gpurun_out/c4v/log.txt 2>&1
for v in "8 0" "8 64" "16 64" "4 64" "16 0"; do
  set -- $v
  if [ "$2" = 0 ]; then unset KP_F16REF_BN; else export KP_F16REF_BN=$2; fi
  echo "workers=$1 bn=$2"
  timeout 600 python bench.py --config C4 --workers $1 --steps 1 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
