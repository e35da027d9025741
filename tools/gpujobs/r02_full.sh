mkdir -p gpurun_out/r02full
exec > gpurun_out/r02full/log.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
