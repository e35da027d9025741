timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
for bn in 128 256; do KP_F16TC_BN=$bn timeout 300 python tools/profile_kernels.py --what msolve_tc --reps 3 > gpurun_out/tc_$bn.log 2>&1; done
KP_F16TC_BN=128 timeout 300 python tools/tensor_profile.py > gpurun_out/tensor_profile2.log 2>&1
timeout 300 python tools/profile_kernels.py --what msolve_tc > gpurun_out/prof_tc_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f16tc -s 2 -c 1 -o gpurun_out/prof_tc2 python tools/profile_kernels.py --what msolve_tc > gpurun_out/ncu_tc2.log 2>&1
tail -n 3 gpurun_out/pytest_tc.log; cat gpurun_out/tc_128.log gpurun_out/tc_256.log gpurun_out/tensor_profile2.log | tail -12
