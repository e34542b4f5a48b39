#!/bin/bash
for l in default variants/la1 variants/la3 variants/la4 variants/la8; do
  if [ $l = default ]; then E=""; else E="NEUROCOMM_B200_LIB=$l/libneurocomm_b200.so"; fi
  echo "$l $(env $E timeout 600 python tools/lif_time.py 2>&1 | tail -1)"
done
