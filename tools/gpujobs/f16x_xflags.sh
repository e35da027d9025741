for x in 0; do
  KP_F16X_XFLAGS=$x timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_f16x" --csv python tools/f16x_time.py 4096 tensor 2>/dev/null | grep gpu__time | awk -F'","' -v x=$x '{print "xflags", x, $NF}' | head -3
done
