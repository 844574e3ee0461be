#!/bin/bash
O=gpurun_out/${TAG:-ktrace}; mkdir -p $O
timeout 300 python tools/ktrace.py > $O/ktrace.log 2>&1
PIPO_WS_DEBUG=128 timeout 300 python tools/ktrace.py c5_out > $O/ktrace_dbg128.log 2>&1
