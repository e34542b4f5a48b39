#!/bin/bash
# LIF pass ILP A/B: persistent-engine phases at config 3 and config 2, per engine variant
mkdir -p gpurun_out
o=gpurun_out/r02_lif_ab.log; : > $o
for l in default variants/lifu1 variants/lifu2 variants/lifu4b4; do
  for n in 10000000 1000000; do
    if [ $l = default ]; then
      r=$(timeout 600 python tools/persistent_phases.py $n 2>&1 | tail -2 | tr '\n' ' ')
    else
      r=$(NEUROCOMM_B200_LIB=$l/libneurocomm_b200.so timeout 600 python tools/persistent_phases.py $n 2>&1 | tail -2 | tr '\n' ' ')
    fi
    echo "$l n=$n: $r" | tee -a $o
  done
done
timeout 600 python tools/push_ncu.py > gpurun_out/r02_push_plain2.json 2>&1; tail -1 gpurun_out/r02_push_plain2.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_deliver_push|k_lif_update" -s 400 -c 2 -o gpurun_out/r02_push2 python tools/push_ncu.py > gpurun_out/r02_push2_ncu.log 2>&1; echo ncu rc=$?
