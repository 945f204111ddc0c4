# N = 2 sweep of the broadcast chunk count (phase times per rank, max over ranks)
for C in 1 4 8 16; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 296$C bench.py --gpus 2 --steps 5 --warmup 3 --bcast-chunks $C --no-e2e --no-cpu > gpurun_out/r25_c$C.json 2> gpurun_out/r25_c$C.err
done
echo done
