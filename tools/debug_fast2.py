import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2501_15021_b200 import akvq as ak, synth as sy
w = sy.LLAVA7B
layer = 2
cfg = ak.make_config(w.U, w.g, w.d, w.G, w.R, w.capacity, w.top_k, 1, ak.AKVQ_BF16)
inp = sy.layer_inputs(w, layer, device="cuda")
res = []
for opt in (0, 1):
    lc = ak.LayerCache(cfg, options=opt)
    lc.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
    di = sy.decode_inputs(w, layer, 0, device="cuda")
    lc.append(di["k"], di["v"], di["types"])
    res.append(lc.decode(di["q"], flags=1).double().cpu().numpy())
a, b = res
print("fast[0,0,:8]   ", np.round(a[0, 0, :8], 4))
print("generic[0,0,:8]", np.round(b[0, 0, :8], 4))
print("ratio", np.round((a / b)[0, 0, :8], 3))
print("diff", np.round((a - b)[0, 0, :16], 4))
