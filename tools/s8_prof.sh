timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_row_g" --launch-skip 4 -c 4 -o gpurun_out/s8_softmax python tools/profile_grouped.py --workload softmax > gpurun_out/s8_ncu.log 2>&1
tail -3 gpurun_out/s8_ncu.log
