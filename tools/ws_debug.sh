python -m paper_2504_03664_b200.build
echo "== movement knobs" > gpurun_out/knobs2.log
for d in 128 131 139 147 155 132 140; do echo "dbg=$d" >> gpurun_out/knobs2.log; PIPO_WS_DEBUG=$d KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_fc2 >> gpurun_out/knobs2.log 2>&1; done
for d in 32 35 43 51; do echo "waits dbg=$d" >> gpurun_out/knobs2.log; PIPO_WS_DEBUG=$d KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv >> gpurun_out/knobs2.log 2>&1; done
