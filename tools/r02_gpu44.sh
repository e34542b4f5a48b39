#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/r02_k5_kernel_ab.log; : > $o
for l in default variants/b4u6 variants/b5u4 variants/b4u6s8 variants/b5u6 variants/b4u8 variants/b4u6; do
  if [ $l = default ]; then r=$(timeout 600 python tools/k5_kernel_ab.py 2>&1 | tail -1)
  else r=$(NEUROCOMM_B200_LIB=$l/libneurocomm_b200.so timeout 600 python tools/k5_kernel_ab.py 2>&1 | tail -1); fi
  echo "$l $r" | tee -a $o
done
