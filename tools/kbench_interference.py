"""Does a concurrent H2D weight stream (as in the live pipeline) slow the decode kernels?
Times pipo_bench_linear with and without a background pinned->device copy loop."""
import sys
import threading
import time

sys.path.insert(0, ".")
import torch

import pipo_synth as synth
from paper_2504_03664_b200 import pipo

pl = pipo.Pipeline(pipo.make_config(synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64), max_batch=4, max_seq=16,
                                    weight_tier=pipo.PIPO_TIER_DEVICE))
cases = [("c5_qkv", 64, 21504, 7168), ("c5_fc2", 64, 7168, 28672)]


def run(tag):
    for name, M, N, K in cases:
        us = pipo.pipo_bench_linear(pl.ctx, 1, pipo.PATH_TM, M, N, K, 10)
        print(tag, name, round(us, 2), flush=True)


run("alone")
stop = False
h = torch.empty(512 << 20, dtype=torch.uint8, pin_memory=True)
d = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def copier():
    with torch.cuda.stream(s):
        while not stop:
            for _ in range(4):
                d.copy_(h, non_blocking=True)
            s.synchronize()


t = threading.Thread(target=copier)
t.start()
time.sleep(0.5)
run("with_h2d")
stop = True
t.join()
