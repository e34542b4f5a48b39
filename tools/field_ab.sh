#!/bin/bash
# A/B of the field term (variants/fieldlop.so = mask + LOP3, variants/fieldmad.so = bit * q IMAD)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do
  bash tools/ab_libs.sh "--steps 1000 --warmup 20 --no-push --no-cpu" variants/fieldmad.so variants/fieldlop.so
  bash tools/ab_libs.sh "--steps 1000 --warmup 20 --no-push --no-cpu" variants/fieldlop.so variants/fieldmad.so
done
bash tools/ab_libs.sh "--steps 1000 --warmup 20 --no-push --no-cpu --tile-words 4096" variants/fieldmad.so variants/fieldlop.so variants/fieldmad.so variants/fieldlop.so
