#!/bin/bash
# GPU session: branch-free tanh (variant tbf) on the tanh patterns, row-group width (chunks
# per thread) on odd softmax widths, ncu hot spots of the column reduce.
mkdir -p gpurun_out
t=s5
bash tools/r4_ab.sh $t "main tbf" "colreduce ln_gelu bert" 0
for c in 32 8 4 2; do
  DISC_ROW_CPT=$c timeout 300 python tools/shape_scan.py softmax "S1=33,65,100,129,255,513,1025" --copies-gb 2 > gpurun_out/${t}_scan_cpt$c.txt 2>&1
done
bash tools/prof_shape.sh colreduce C=1024,N=1000000 "k_col" ${t}_col
DISC_LIB_VARIANT=tbf bash tools/prof_shape.sh colreduce C=1024,N=1000000 "k_col" ${t}_col_tbf
