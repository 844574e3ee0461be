# launcher check: 2 ranks sharing the one GPU (self-launch and torchrun), c2 batch-shard + sharded-streaming variant
mkdir -p gpurun_out/n2
timeout 900 python bench.py --gpus 2 --allow-shared-gpu --config c2 --steps 3 --warmup 3 > gpurun_out/n2/self.json 2> gpurun_out/n2/self.err; echo self rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --allow-shared-gpu --config c2 --steps 3 --warmup 3 > gpurun_out/n2/torchrun.json 2> gpurun_out/n2/torchrun.err; echo torchrun rc=$?
timeout 600 python bench.py --gpus 2 --impl reference --steps 1 --warmup 0 > gpurun_out/n2/ref.json 2> gpurun_out/n2/ref.err; echo ref rc=$?
# decode attention isolated: TLB-warm (one K/V copy) vs TLB-cold (rotating over 16 / 40 GB)
for mb in 384 16384 40000 384; do
  PIPO_BENCH_KV_MB=$mb timeout 300 python tools/abench.py c5 c6 2>&1 | sed "s/^/kvmb=$mb /" >> gpurun_out/n2/abench_tlb.log
done
