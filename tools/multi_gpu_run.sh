set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r24_topo.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider > gpurun_out/r24_dist.log 2>&1
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_C3_n${N}_r02.json 2> gpurun_out/bench_C3_n${N}_r02.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 4 --steps 5 --warmup 3 --bcast-chunks 1 --no-e2e --no-cpu > gpurun_out/bench_C3_n4_chunks1_r02.json 2> gpurun_out/bench_C3_n4_chunks1_r02.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 3 --warmup 3 --config C5 --no-e2e > gpurun_out/bench_C5_n${N}_r02.json 2> gpurun_out/bench_C5_n${N}_r02.err
done
mkdir -p profiles/r02
cp gpurun_out/bench_C3_n2_r02.json gpurun_out/bench_C3_n4_r02.json gpurun_out/bench_C5_n2_r02.json gpurun_out/bench_C5_n4_r02.json profiles/r02/
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --proxy-gpus 8 --no-e2e --no-cpu > gpurun_out/bench_C3_proxy8_r02.json 2> gpurun_out/proxy.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --proxy-gpus 8 --config C5 --steps 3 --no-e2e --no-cpu > gpurun_out/bench_C5_proxy8_r02.json 2>> gpurun_out/proxy.err
echo done
