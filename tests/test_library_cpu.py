"""CPU-side checks of the C-ABI library (-m "not gpu"): it builds for sm_100a, loads,
exports every symbol include/akvq.h declares, and its host-only arithmetic (config
validation, layout, memory report) is right.  No kernel is launched here."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ak():
    from paper_2501_15021_b200 import akvq, build
    if not os.path.exists(akvq.LIB_PATH):
        build.build()
    akvq.lib()
    return akvq


def test_exports_match_header(ak):
    hdr = open(os.path.join(ROOT, "include", "akvq.h")).read()
    declared = set(re.findall(r"^[a-z_ ]*\*?\s*(akvq_[a-z_]+)\s*\(", hdr, re.M))
    assert declared == set(ak.EXPORTS), declared ^ set(ak.EXPORTS)
    raw = C.CDLL(ak.LIB_PATH)
    for name in declared:
        assert hasattr(raw, name), name
    assert "sm_100a" in ak.version()
    assert ak.status_str(ak.AKVQ_ECAPACITY) == "capacity exceeded"


def test_sass_is_sm100a(ak):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ak.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _cfg(ak, **kw):
    base = dict(U=4, g=1, d=128, G=128, R=32, capacity=800, top_k=15, kind=ak.AKVQ_PSA)
    base.update(kw)
    return ak.make_config(base["U"], base["g"], base["d"], base["G"], base["R"],
                          base["capacity"], base["top_k"], base["kind"])


def test_config_validation(ak):
    assert ak.akvq_cache_bytes(_cfg(ak)) > 0
    bad = {  # S:395 power-of-two guard etc. -> EINVAL; unbuilt shapes -> EUNSUPPORTED
        ak.AKVQ_EINVAL: [dict(d=96), dict(G=48), dict(U=0), dict(R=-1), dict(capacity=0),
                         dict(top_k=-1), dict(kind=5)],
        ak.AKVQ_EUNSUPPORTED: [dict(d=256), dict(G=16), dict(d=64, G=128), dict(top_k=33),
                               dict(g=17)],
    }
    for st, cases in bad.items():
        for kw in cases:
            with pytest.raises(ak.AkvqError) as e:
                ak.akvq_cache_layout(_cfg(ak, **kw))
            assert e.value.status == st, kw
            assert ak.akvq_cache_bytes(_cfg(ak, **kw)) == 0
    c = _cfg(ak)
    c.clip2 = 0.0
    with pytest.raises(ak.AkvqError):
        ak.akvq_cache_layout(c)


def test_layout_arithmetic(ak):
    y = ak.akvq_cache_layout(_cfg(ak))
    d = G = 128
    assert y.cap == 896 and y.n_pages == 7 and y.slots == 160 and y.ng == 1
    # one page = 80 bytes per token at d = G = 128: codes 2x32 + meta 16
    assert y.page_bytes == 128 * (32 + 32 + 8 + 8)
    assert y.bitmask_words == 896 // 32 and y.side_cap == 15 and y.side_entry_bytes == 4 * d
    offs = [y.pages_off, y.ring_off, y.bitmask_off, y.side_idx_off, y.side_cnt_off, y.side_off]
    assert offs == sorted(offs) and all(o % 256 == 0 for o in offs)
    assert y.ring_off >= 4 * 7 * y.page_bytes
    t = ak.akvq_cache_layout(_cfg(ak, kind=ak.AKVQ_TSA))
    assert t.side_cap == 896 and t.side_entry_bytes == 144          # d/2*2 + 16*ng


def _host_cache(ak, cfg, L, n_q):
    c = ak.akvq_cache()
    c.cfg = cfg
    c.lay = ak.akvq_cache_layout(cfg)
    c.L, c.n_q = L, n_q
    return c


def test_memory_report_closed_forms(ak):
    # pure int2, head_dim 128, group 128 -> 2.5 bits, ratio 6.4
    cfg = _cfg(ak, R=0, top_k=0, capacity=1024)
    r = ak.akvq_memory_report(_host_cache(ak, cfg, 1024, 1024), 0)
    assert r.effective_bits_per_element == pytest.approx(2.5, abs=1e-12)
    assert r.compression_ratio_vs_fp16 == pytest.approx(6.4, abs=1e-12)
    # all 16-bit (window covers everything) -> 16 bits, ratio 1
    r = ak.akvq_memory_report(_host_cache(ak, _cfg(ak, R=512, capacity=512), 300, 0), 0)
    assert r.effective_bits_per_element == pytest.approx(16.0)
    # S:432-style mixed PSA layer: 128 quantized (1 pivot) + 172 ring tokens
    r = ak.akvq_memory_report(_host_cache(ak, _cfg(ak, R=172, capacity=300, top_k=1), 300, 128), 1)
    # closed form: 16-bit rows 173 tokens; 2-bit codes for 127 tokens; meta = K 8 B per
    # channel per block (1 block) + V 8 B per token over 128 tokens
    total_bits = 173 * 2 * 128 * 16 + 127 * 2 * 128 * 2 + (128 * 8 + 128 * 8) * 8
    assert r.effective_bits_per_element == pytest.approx(total_bits / (300 * 2 * 128), rel=1e-12)
    # asymptote -> 2.5
    big = _cfg(ak, R=128, capacity=100000, top_k=15)
    n_q = (100000 - 128) // 128 * 128
    r = ak.akvq_memory_report(_host_cache(ak, big, 100000, n_q), 15)
    assert abs(r.effective_bits_per_element - 2.5) < 0.05


def test_memory_report_tsa_needs_the_text_count(ak):
    """A TSA layer's 4-bit text rows are counted from the caller's side
    count; -1 (unknown, the count lives on the device) is rejected."""
    cfg = _cfg(ak, kind=ak.AKVQ_TSA, R=172, capacity=300)
    c = _host_cache(ak, cfg, 300, 128)
    with pytest.raises(ak.AkvqError) as e:
        ak.akvq_memory_report(c, -1)
    assert e.value.status == ak.AKVQ_EINVAL
    r = ak.akvq_memory_report(c, 100)
    d = 128
    assert r.bytes_int4 == pytest.approx(4 * 100 * 2 * (d / 2 + 8))
    assert r.bytes_int2 == pytest.approx(4 * 28 * 2 * d / 4)
    assert r.bytes_fp16 == pytest.approx(4 * 172 * 2 * d * 2)
    with pytest.raises(ak.AkvqError):
        ak.akvq_memory_report(c, 129)                   # more side rows than n_q


@pytest.mark.parametrize("g", [1, 2, 7, 16])
def test_ticket_region_covers_every_head_group(ak, g):
    """The merge-ticket region holds one ticket per (unit, GQA head group) of the
    decode kernel for every supported q_per_kv (g up to 16)."""
    y = ak.akvq_cache_layout(_cfg(ak, g=g))
    assert y.total_bytes - y.ticket_off >= 4 * 4 * max(1, g)      # U = 4 units, <= g groups


def test_exact_r_config(ak):
    """exact_r (R26) needs per-token K and is 0 / 1; the layout does not change."""
    def mk(k_axis, exact_r):
        return ak.make_config(4, 1, 128, 128, 32, 800, 15, ak.AKVQ_PSA, ak.AKVQ_BF16, 0.8, 1.0,
                              k_axis, exact_r=exact_r)
    for k_axis, ex in ((0, 1), (1, 2), (1, -1)):
        with pytest.raises(ak.AkvqError) as e:
            ak.akvq_cache_layout(mk(k_axis, ex))
        assert e.value.status == ak.AKVQ_EINVAL, (k_axis, ex)
    assert ak.akvq_cache_bytes(mk(1, 1)) == ak.akvq_cache_bytes(mk(1, 0)) > 0
