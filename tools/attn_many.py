import sys, time
sys.path.insert(0, ".")
import numpy as np
from tests.gpu_util import pipo_mod, rel_inf
from oracle import opt
pipo = pipo_mod()
import pipo_synth as synth
shape = synth.OPTShape(d_model=256, n_layers=1, n_heads=4, ffn_dim=512, vocab=512, max_pos=64)
pl = pipo.Pipeline(pipo.make_config(shape, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE))
for (b, n, past, d, H) in [(int(x) for x in c.split(",")) for c in sys.argv[1:]]:
    rng = np.random.default_rng(n + d)
    q = (rng.standard_normal((b, n, d)) * (d // H) ** -0.5).astype(np.float16)
    L = past + n
    k = rng.standard_normal((L, b, d)).astype(np.float16)
    v = rng.standard_normal((L, b, d)).astype(np.float16)
    t0 = time.time()
    o = pipo.pipo_attention_prefill(pl.ctx, q, k, v, past, H, 0)
    print((b, n, past, d, H), "done in %.2fs" % (time.time() - t0), flush=True)
    ref = opt.attention(q.astype(np.float64), k.astype(np.float64).transpose(1, 0, 2), v.astype(np.float64).transpose(1, 0, 2), past, H)
    print("   rel err", rel_inf(o, ref), flush=True)
