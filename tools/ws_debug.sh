python -m paper_2504_03664_b200.build
for dbg in 0 1 2 4 3 7; do echo "dbg=$dbg"; PIPO_WS_DEBUG=$dbg timeout 120 python tools/kbench.py c5_qkv c2_qkv 2>&1 | grep -o '"ws": {[^}]*}' ; done > gpurun_out/ws_debug.log 2>&1
