"""HBM -> shared memory streaming with cp.async.bulk, one CTA per SM: GB/s by request
size x ring depth, and with each CTA's requests spread over several streams (regions)."""
import sys
sys.path.insert(0, ".")
import pipo_synth as synth
from paper_2504_03664_b200 import pipo
pl = pipo.Pipeline(pipo.make_config(synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64), max_batch=4, max_seq=16,
                                    weight_tier=pipo.PIPO_TIER_DEVICE))
for streams in (1, 2, 4):
    for chunk in (4352, 8704, 17408, 34816):
        row = []
        for stages in (2, 4, 6, 8, 12, 16):
            if chunk * stages > 220 * 1024:
                continue
            row.append(f"{stages}:{pipo.pipo_probe_bulk(pl.ctx, chunk, stages, streams):.0f}")
        print(f"streams {streams} chunk {chunk}", " ".join(row), flush=True)
