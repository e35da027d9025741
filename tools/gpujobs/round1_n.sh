# bench lines for C1-C4 + reference arm sanity at C1
for c in C1 C2 C3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_n_$c.json 2> gpurun_out/bench_n_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config C4 --warmup 3 > gpurun_out/bench_n_C4.json 2> gpurun_out/bench_n_C4.err; echo "C4 rc=$?"
timeout 600 python bench.py --impl reference --config C1 --steps 2 --warmup 1 > gpurun_out/bench_n_ref_C1.json 2> gpurun_out/bench_n_ref_C1.err; echo "refC1 rc=$?"
for f in gpurun_out/bench_n_*.json; do echo $f; cut -c1-400 $f; done
