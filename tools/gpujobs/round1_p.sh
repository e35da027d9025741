# f16ref UNIT=64 sweep, pipe-mix microbench, GPU tests (incl. concurrency), C4 bench with workers
cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix mix.cu && ./mix > ../../gpurun_out/mix.txt 2>&1; cd ../..
cat gpurun_out/mix.txt
timeout 900 python tools/sweep_f16ref.py 0 1 5 6 > gpurun_out/sweep_p.txt 2>&1; cat gpurun_out/sweep_p.txt
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_p.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/pytest_p.log
for w in 1 4; do timeout 900 python bench.py --config C4 --workers $w > gpurun_out/bench_p_c4_w$w.json 2>gpurun_out/bench_p_c4_w$w.err; echo "C4 w=$w rc=$?"; cut -c1-330 gpurun_out/bench_p_c4_w$w.json; done
