# banded operator: generic vs tap-specialised kernels, pass-A register caps
exec > gpurun_out/band/log.txt 2>&1; set -x
python -c "import __graft_entry__ as g; g.build()"
KP_BAND_GENERIC=1 timeout 300 python tools/time_op.py 2>&1 | tail -1
timeout 300 python tools/time_op.py 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"band_" --csv --log-file gpurun_out/band/spec.csv python tools/time_op.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/band/spec.csv
KP_BAND_GENERIC=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"band_" --csv --log-file gpurun_out/band/gen.csv python tools/time_op.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/band/gen.csv
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_configs.py -q -m gpu -x -k "band or operator or kronsum" 2>&1 | tail -2
for fl in "-DKP_BAND_A_MINB=3" "-DKP_BAND_A_MINB=5"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Xptxas -v $fl -c paper_2311_15393_b200/csrc/banded.cu -o paper_2311_15393_b200/_build/banded.cu.o 2>&1 | grep -A2 "band_cols_kernelILi41" | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores"
  python -c "import __graft_entry__ as g; g.build()"
  echo "variant $fl"; timeout 300 python tools/time_op.py 2>&1 | tail -1
done
