# Real 1/2/4-GPU bench lines (C3, C5) and the labelled 8-GPU proxies; the 2/4-GPU
# lines are copied to profiles/r02/ for the proxy's overhead extrapolation.
set -x
mkdir -p gpurun_out profiles/r02
timeout 600 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider > gpurun_out/r32_dist.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C3_n1_r02.json 2> gpurun_out/bench_C3_n1_r02.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_C3_n${N}_r02.json 2> gpurun_out/bench_C3_n${N}_r02.err
done
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 3 --warmup 3 --config C5 --no-e2e > gpurun_out/bench_C5_n${N}_r02.json 2> gpurun_out/bench_C5_n${N}_r02.err
done
cp gpurun_out/bench_C3_n2_r02.json gpurun_out/bench_C3_n4_r02.json gpurun_out/bench_C5_n2_r02.json gpurun_out/bench_C5_n4_r02.json profiles/r02/
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --proxy-gpus 8 --no-e2e --no-cpu > gpurun_out/bench_C3_proxy8_r02.json 2> gpurun_out/proxy.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --proxy-gpus 8 --config C5 --steps 3 --no-e2e --no-cpu > gpurun_out/bench_C5_proxy8_r02.json 2>> gpurun_out/proxy.err
echo done
