"""Debug: compare dp4a page path vs generic path vs oracle on a 7B layer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2501_15021_b200 import akvq as ak, synth as sy
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from parity import f16_bits

w = sy.LLAVA7B
for layer in (0, 2):
    kind = w.kind(layer)
    cfg = ak.make_config(w.U, w.g, w.d, w.G, w.R, w.capacity, w.top_k, kind, ak.AKVQ_BF16)
    inp = sy.layer_inputs(w, layer, device="cuda")
    outs = []
    for opt in (0, 1):
        lc = ak.LayerCache(cfg, options=opt)
        lc.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
        di = sy.decode_inputs(w, layer, 0, device="cuda")
        lc.append(di["k"], di["v"], di["types"])
        for flags in (0, 1):
            outs.append(lc.decode(di["q"], flags=flags).double().cpu().numpy())
    oc = oracle.OracleCache(oracle.OracleConfig(w.U, w.g, w.d, w.G, w.R, w.capacity, w.top_k, kind, oracle.BF16))
    oc.prefill(f16_bits(inp["K"]), f16_bits(inp["V"]), inp["types"].cpu().numpy(), inp["colsum"].cpu().numpy())
    oc.append(f16_bits(di["k"]), f16_bits(di["v"]), di["types"].cpu().numpy())
    ref = oc.decode(f16_bits(di["q"]))
    refr = oc.decode(f16_bits(di["q"]), out_rotated=True)
    for name, o, r in (("fast", outs[0], ref), ("fast-rot", outs[1], refr), ("generic", outs[2], ref), ("generic-rot", outs[3], refr)):
        e = np.abs(o - r)
        u, h, c = np.unravel_index(e.argmax(), e.shape)
        print(f"layer {layer} {name:12s} max {e.max():.2e} at unit {u} ch {c}; mean {e.mean():.2e}; "
              f"units>1e-3: {sorted(set(np.nonzero(e.max(axis=(1,2)) > 1e-3)[0].tolist()))[:10]}")
    e = np.abs(outs[1] - refr)[..., :]
    print("  per-channel max err (fast-rot) unit worst:", np.round(e.max(axis=(0,1)).reshape(8,16).max(1), 5))
