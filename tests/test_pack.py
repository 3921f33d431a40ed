"""Host packer (pack.py) vs the golden W: evaluate the segment closed form in
exact Python integers (test-only restatement of the device formula) and
compare with the reference's weights bit for bit.  Runs on CPU."""

from fractions import Fraction

import pytest

from helpers import own_problem

from paper_2311_15566_b200 import pack
from paper_2311_15566_b200.domain import natural_key


def eval_w(row_ptr, segs, K, cfg, L, wide=False):
    D, P, M = cfg.data_parallel, cfg.pipeline_stages, cfg.tensor_shards
    cols = []
    for d in range(D):
        for p in range(P):
            for m in range(M):
                q, r = divmod(L, P)
                s0 = p * q + min(p, r)
                s1 = s0 + q + (1 if p < r else 0)
                w = K // M
                cols.append((d + 1, s0, s1, m * w, m * w + w))
    if wide:  # two SEGMENT slots per sk_segment_wide; row_ptr counts slots
        segs = segs.view(pack.SEGMENT_WIDE)
        row_ptr = row_ptr // 2
    W = []
    for i in range(len(row_ptr) - 1):
        row = []
        for d, s0, s1, i0, i1 in cols:
            acc = 0
            for s in segs[row_ptr[i]:row_ptr[i + 1]]:
                ol = min(int(s["l1"]), s1) - max(int(s["l0"]), s0)
                oi = min(int(s["b"]), i1) - max(int(s["a"]), i0)
                if ol <= 0 or oi <= 0 or (s["pipe"] != 0 and s["pipe"] != d):
                    continue
                acc += ol * oi * int(s["unit"])
            row.append(float(Fraction(acc, K)))
        W.append(row)
    return W


@pytest.mark.parametrize("name", ["mapping", "scenario", "edge"])
def test_segments_reproduce_golden_weights(golden, name):
    doc = golden(name)
    cases = doc["cases"] if name != "scenario" else doc["maps"]
    checked = wide_seen = 0
    for case in cases:
        if "W" not in case:
            continue
        model, cfg, G, insts, inh, rq, fw = own_problem(case)
        invs = [inv for inst in sorted(insts, key=lambda i: natural_key(i.id))
                for inv in inst.gpu_inventories]
        K = pack.common_denominator(invs, cfg.tensor_shards)
        need = pack.need_tokens(pack.inherited_by_new(inh, rq), cfg.data_parallel)
        row_ptr, segs, wide = pack.pack_rows(invs, K, model.bytes_per_layer,
                                             model.kv_bytes_per_token_per_layer, need)
        W = eval_w(row_ptr, segs, K, cfg, model.num_layers, wide)
        assert [[x.hex() for x in row] for row in W] == case["W"]
        # the native packer (csrc/hostpack.cpp) equals the Python statement
        assert K == pack.py_common_denominator(invs, cfg.tensor_shards)
        rp2, sg2, w2 = pack.py_pack_rows(invs, K, model.bytes_per_layer,
                                         model.kv_bytes_per_token_per_layer, need)
        assert w2 == wide
        assert rp2.tobytes() == row_ptr.tobytes() and sg2.tobytes() == segs.tobytes()
        # forcing the general-range encoding keeps the weights
        rp3, sg3, w3 = pack.pack_rows(invs, K, model.bytes_per_layer,
                                      model.kv_bytes_per_token_per_layer, need, wide=True)
        assert w3
        W3 = eval_w(rp3, sg3, K, cfg, model.num_layers, True)
        assert [[x.hex() for x in row] for row in W3] == case["W"]
        checked += 1
        wide_seen += wide
    assert checked >= 10
    if name == "edge":
        assert wide_seen >= 10   # numerators >= 2^53 and K > 2^31 - 1 take the wide encoding


def test_structured_row_is_one_model_and_one_cache_segment():
    inv_m = tuple((layer, Fraction(1, 4), Fraction(2, 4)) for layer in range(3, 9))
    inv_c = tuple((f"r{j}", layer, Fraction(1, 4), Fraction(2, 4), 600 + j)
                  for j in range(4) for layer in range(3, 9))
    from paper_2311_15566_b200.domain import ContextInventory

    inv = ContextInventory(inv_m, inv_c)
    need = {f"r{j}": [(1, 600 + j)] for j in range(4)}
    segs = pack.pack_row(inv, 8, 1000, 16, need)
    rp, sg, wide = pack.pack_rows([inv], 8, 1000, 16, need)
    assert not wide
    assert sg.tolist() == [(3, 9, 2, 4, 0, 0, 1000), (3, 9, 2, 4, 1, 0, 16 * (600 + 601 + 602 + 603))]
    assert segs == [(3, 9, 2, 4, 0, 1000), (3, 9, 2, 4, 1, 16 * (600 + 601 + 602 + 603))]
