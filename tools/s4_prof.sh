mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:_g" --launch-skip 3 -c 3 -o gpurun_out/s4_lngelu python tools/profile_grouped.py --workload ln_gelu > gpurun_out/s4_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:_g" --launch-skip 4 -c 4 -o gpurun_out/s4_softmax python tools/profile_grouped.py --workload softmax >> gpurun_out/s4_ncu.log 2>&1
tail -5 gpurun_out/s4_ncu.log
