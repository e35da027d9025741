mkdir -p gpurun_out/r02c4
exec > gpurun_out/r02c4/log.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x 2>&1 | tail -3
timeout 1200 python bench.py --config C4 --no-cpu-baseline > gpurun_out/r02c4/C4.json 2> gpurun_out/r02c4/C4.err
python -c "
import json; d=json.load(open('gpurun_out/r02c4/C4.json')); print('C4', d['value'], d['e2e']['value'], d['gpu_launches'], d['roofline']['ms_per_launch'], d.get('tensor_mode',{}).get('value'))"
timeout 900 python tools/c4_timeline.py > gpurun_out/r02c4/tl2.txt 2>&1
grep -v Warn gpurun_out/r02c4/tl2.txt | head -4; grep -A3 "idle gaps" gpurun_out/r02c4/tl2.txt
