for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n > gpurun_out/strong_n$n.json 2> gpurun_out/strong_n$n.err; echo "n=$n rc=$?"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --impl reference > gpurun_out/strong_ref_n4.json 2> gpurun_out/strong_ref_n4.err; echo "ref rc=$?"
