#!/bin/bash
# ncu --set full of the column reduce and an odd-width softmax epilogue: pipes and stalls.
mkdir -p gpurun_out
t=s9
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_col_g|k_col\b|k_col<" -c 1 -f -o /tmp/${t}_col \
  python tools/profile_one.py --workload colreduce --shape C=1024,N=1000000 --reps 1 > gpurun_out/${t}_col_run.log 2>&1
python tools/ncu_pipes.py /tmp/${t}_col.ncu-rep > gpurun_out/${t}_col_pipes.txt 2>&1
python tools/ncu_summary.py /tmp/${t}_col.ncu-rep > gpurun_out/${t}_col_summary.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_row" -c 2 -f -o /tmp/${t}_sm33 \
  python tools/profile_one.py --workload softmax --shape S0=646464,S1=33 --reps 1 > gpurun_out/${t}_sm33_run.log 2>&1
python tools/ncu_pipes.py /tmp/${t}_sm33.ncu-rep > gpurun_out/${t}_sm33_pipes.txt 2>&1
python tools/ncu_summary.py /tmp/${t}_sm33.ncu-rep > gpurun_out/${t}_sm33_summary.txt 2>&1
cp /tmp/${t}_col.ncu-rep gpurun_out/ 2>/dev/null
