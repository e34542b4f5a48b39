#!/bin/bash
# A/B of the field term: variants/flop.so (sign mask + LOP3, ALU) vs variants/ffma.so (mul.hi + mad, FMA pipe)
for r in 1 2; do
  bash tools/ab_libs.sh "--steps 1000 --warmup 20 --no-push --no-cpu" variants/ffma.so variants/flop.so
  bash tools/ab_libs.sh "--steps 1000 --warmup 20 --no-push --no-cpu" variants/flop.so variants/ffma.so
done
bash tools/ab_libs.sh "--steps 1000 --warmup 20 --no-push --no-cpu --tile-words 4096" variants/ffma.so variants/flop.so variants/ffma.so variants/flop.so
