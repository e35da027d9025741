# full ncu capture of both banded passes at C5 size + SASS instruction mix
exec > gpurun_out/band/ncu_log.txt 2>&1
rm -f gpurun_out/band/full.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"band_" -s 2 -c 2 -o gpurun_out/band/full python tools/time_op.py > /dev/null 2>&1
python tools/ncu_keys.py gpurun_out/band/full.ncu-rep
python tools/sass_mix.py gpurun_out/band/full.ncu-rep band_cols 12
python tools/sass_mix.py gpurun_out/band/full.ncu-rep band_rows 12
