mkdir -p gpurun_out/r02q
exec > gpurun_out/r02q/log.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4; echo "pytest rc=$?"
for ks in 0 1; do
  if [ $ks = 1 ]; then export KP_F16REF_KSPLIT=1; fi
  for c in C1; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-other-runs --no-tensor > gpurun_out/r02q/${c}_$ks.json 2> gpurun_out/r02q/${c}_$ks.err; python -c "
import json; d=json.load(open('gpurun_out/r02q/${c}_$ks.json')); print('$c ksplit-off=$ks', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'])"; done
done
