import numpy as np, sys
sys.path.insert(0, '.')
from tests import q17b_model as qm
from tests.gpu_util import load_masters, pipo_mod
from oracle import opt
pipo = pipo_mod()
emb, layers = qm.masters()
b = 2
np.set_printoptions(precision=4, suppress=True, linewidth=150)
for kv_fmt in ("fp16", "int4"):
    q4 = kv_fmt == "int4"
    ref = opt.OracleOPT.from_masters(1, emb, layers, "int4", 4, kv_int4=q4)
    ref.prefill(qm.prompt(b)); pre = ref.capture[0][:, 0].copy()
    ref.decode(qm.decode_tokens(b)); want = ref.capture[0][:, 0]
    cfg = pipo.make_config(qm.SHAPE, max_batch=b, max_seq=4, weight_tier=pipo.PIPO_TIER_HOST,
                           kv_fmt=pipo.PIPO_W_INT4_G64 if q4 else pipo.PIPO_W_FP16)
    with pipo.Pipeline(cfg) as pl:
        load_masters(pl, emb, layers)
        cap0 = np.zeros((1, b, 1, 64), np.float32)
        pipo.pipo_debug_capture(pl.ctx, cap0)
        pl.prefill(qm.prompt(b))
        cap = np.zeros((1, b, 1, 64), np.float32)
        pipo.pipo_debug_capture(pl.ctx, cap)
        pl.decode_step(qm.decode_tokens(b))
    print(kv_fmt, "prefill err", np.abs(cap0[0][:, 0] - pre).max(), "decode err", np.abs(cap[0][:, 0] - want).max())
    print(" got ", cap[0][0, 0, :12]); print(" want", want[0, :12]); print(" pre got", cap0[0][0,0,:8], "want", pre[0,:8])
