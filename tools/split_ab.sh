for s in 0 1 2; do
  echo "split=$s"; NC_BLOCK_SPLIT=$s bash tools/strong_tiles.sh 4 "16384 auto"
done
for s in 0 1; do echo "split=$s"; NC_BLOCK_SPLIT=$s bash tools/strong_tiles.sh 2 "auto"; done
for s in 0 1; do echo "split=$s N=1"; NC_BLOCK_SPLIT=$s python bench.py --steps 500 --warmup 10 --no-push --no-cpu 2>/dev/null | tail -n 1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'])"; done
