"""Pin the CPU oracle (oracle/ulysses_oracle.py) before trusting it.

Every check compares the restatement against vectors produced by the
unmodified reference (tests/golden/*.npz, made by oracle/gen_golden.py)
or against the reference's own known answers (cited test file:line).
"""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import ulysses_oracle as O


def load(name):
    return np.load(os.path.join(GOLDEN, name))


class TestAllToAllGolden:
    def test_block_transpose_known_answer(self):
        # test_simgroup.py:143-151
        g = load("a2a.npz")
        out = O.all_to_all([np.array([0.0, 1.0]), np.array([10.0, 11.0])], 0, 0)
        assert np.array_equal(out[0], g["transpose2_r0"]) and np.array_equal(out[0], [0.0, 10.0])
        assert np.array_equal(out[1], g["transpose2_r1"]) and np.array_equal(out[1], [1.0, 11.0])

    @pytest.mark.parametrize("ci", range(8))
    def test_cases_bitwise(self, ci):
        g = load("a2a.npz")
        meta = g[f"case{ci}_meta"]
        p, split, concat, agg, egress = (int(x) for x in meta[:5])
        ins = [g[f"case{ci}_in{r}"] for r in range(p)]
        outs = O.all_to_all(ins, split, concat)
        for r in range(p):
            exp = g[f"case{ci}_out{r}"]
            assert outs[r].dtype == np.float32
            assert outs[r].tobytes() == exp.tobytes()
        assert O.all_to_all_metering(ins[0].size, p) == (agg, egress)

    def test_metering_known_answer(self):
        # test_simgroup.py:153-164: (8,2,8) local at P=4 -> egress 96
        assert O.all_to_all_metering(8 * 2 * 8, 4) == (4 * 128, 96)

    def test_self_inverse_and_conservation(self):
        # test_simgroup.py:166-187
        xs = [np.random.default_rng([7, r]).standard_normal((4, 2, 6)) for r in range(2)]
        back = O.all_to_all(O.all_to_all(xs, 2, 0), 0, 2)
        assert all(np.array_equal(a, b) for a, b in zip(xs, back))
        ys = O.all_to_all(xs, 0, 1)
        assert np.array_equal(np.sort(np.concatenate([x.ravel() for x in xs])),
                              np.sort(np.concatenate([y.ravel() for y in ys])))

    def test_shard_error(self):
        with pytest.raises(O.ShardError):
            O.all_to_all([np.zeros((3, 2))] * 2, 0, 1)

    def test_head_slice_spec(self):
        # test_ulysses.py:81-94: rank r's head shard == split_heads(x)[:, :, rH/P:(r+1)H/P]
        x = O.make_tensor((8, 1, 4, 2), 2, 0)
        p = 2
        res = O.seq_to_head([x[r * 4:(r + 1) * 4] for r in range(p)], 4)
        for r in range(p):
            assert np.array_equal(res[r], x[:, :, r * 2:(r + 1) * 2, :])

    def test_volume_plugins(self):
        # test_costmodel.py:26-28, 36-44
        assert O.ulysses_volume(1024, 1, 512, 4, "paper_asymptotic") == 524288
        assert O.ulysses_volume(8, 1, 8, 4, "exact") == 48
        assert O.ulysses_volume(8, 1, 8, 1, "exact") == 0


class TestSoftmaxKnownAnswers:
    def test_single_entry_and_causal_first(self):
        # test_tensor.py:72-77
        assert np.array_equal(O.row_softmax(np.array([[3.7]]), "none"), [[1.0]])
        assert np.array_equal(O.row_softmax(np.zeros((1, 3)), "causal"), [[1.0, 0.0, 0.0]])

    def test_hand_exp(self):
        # test_tensor.py:79-85
        x = [1.0, 2.0, 3.0]
        e = [math.exp(v - 3.0) for v in x]
        assert np.allclose(O.row_softmax(np.array([x]), "none")[0], [v / sum(e) for v in e],
                           rtol=0, atol=1e-15)

    def test_masked_exactly_zero_and_offsets(self):
        # test_tensor.py:95-122
        out = O.row_softmax(np.ones((4, 4)), "causal")
        assert np.array_equal(out[0, 1:], np.zeros(3))
        s = np.random.default_rng(3).standard_normal((8, 8))
        full = O.row_softmax(s, "causal")
        parts = [O.row_softmax(s[i:i + 2], "causal", row_offset=i) for i in range(0, 8, 2)]
        assert np.array_equal(full, np.concatenate(parts, 0))

    def test_lse_consistent_with_softmax(self):
        s = np.random.default_rng(5).standard_normal((6, 6)) * 3
        lse = O.row_lse(s, "causal")
        p = O.row_softmax(s, "causal")
        vis = O.visibility("causal", 6, 6)
        np.testing.assert_allclose(np.where(vis, np.exp(s - lse[:, None]), 0.0), p,
                                   rtol=0, atol=1e-15)

    def test_matmul_exact_vs_naive(self):
        # test_tensor.py:54-63
        rng = np.random.default_rng(1)
        a, b = rng.standard_normal((5, 7)), rng.standard_normal((7, 3))
        naive = np.zeros((5, 3))
        for i in range(5):
            for j in range(3):
                acc = 0.0
                for k in range(7):
                    acc += a[i, k] * b[k, j]
                naive[i, j] = acc
        assert np.array_equal(O.matmul(a, b), naive)


class TestKernelKnownAnswers:
    def test_single_token_is_v(self):
        # test_kernels.py:32-35
        rng = np.random.default_rng(0)
        q, k, v = (rng.standard_normal((1, 2, 4)) for _ in range(3))
        c, _ = O.attention_head(q, k, v, "none", 0.5)
        assert np.array_equal(c, v)

    def test_causal_first_row_is_v0(self):
        # test_kernels.py:37-40
        rng = np.random.default_rng(2)
        q, k, v = (rng.standard_normal((5, 1, 3)) for _ in range(3))
        c, _ = O.attention_head(q, k, v, "causal", 0.7)
        assert np.allclose(c[0], v[0], rtol=0.0, atol=1e-15)

    def test_backward_finite_differences(self):
        # test_kernels.py:105-131
        n, b, hd = 5, 1, 3
        rng = np.random.default_rng(9)
        q, k, v = (rng.standard_normal((n, b, hd)) for _ in range(3))
        scale = 1.0 / np.sqrt(hd)
        out, _ = O.attention_head(q, k, v, "causal", scale)
        dq, dk, dv = O.attention_head_backward(q, k, v, 2.0 * out, "causal", scale)

        def loss(q, k, v):
            return float((O.attention_head(q, k, v, "causal", scale)[0] ** 2).sum())

        eps = 1e-6
        r = np.random.default_rng(1)
        for name, arr, grad in (("q", q, dq), ("k", k, dk), ("v", v, dv)):
            for _ in range(5):
                i, j, l = r.integers(n), r.integers(b), r.integers(hd)
                hi, lo = arr.copy(), arr.copy()
                hi[i, j, l] += eps
                lo[i, j, l] -= eps
                args_hi = {"q": q, "k": k, "v": v} | {name: hi}
                args_lo = {"q": q, "k": k, "v": v} | {name: lo}
                fd = (loss(**args_hi) - loss(**args_lo)) / (2 * eps)
                assert abs(grad[i, j, l] - fd) <= 1e-6 * max(1.0, abs(grad[i, j, l]), abs(fd))

    def test_blas_mode_matches_exact(self):
        rng = np.random.default_rng(4)
        q, k, v = (rng.standard_normal((40, 1, 16)) for _ in range(3))
        a, la = O.attention_head(q, k, v, "causal", 0.25, exact=True)
        b, lb = O.attention_head(q, k, v, "causal", 0.25, exact=False)
        assert np.abs(a - b).max() <= 1e-12 and np.abs(la - lb).max() <= 1e-12


class TestUlyssesGolden:
    @pytest.mark.parametrize("ci", range(4))
    def test_small_cases(self, ci):
        g = load("attn_small.npz")
        p, n, b, h, hd, causal, seed = (int(x) for x in g[f"case{ci}_meta"])
        kind = "causal" if causal else "none"
        q, k, v, do = (g[f"case{ci}_{t}"].astype(np.float64) for t in ("q", "k", "v", "do"))
        # inputs are the seeded generator's output (regenerable on the GPU box)
        assert np.array_equal(q, O.make_tensor((n, b, h, hd), seed, 1))
        nl = n // p
        sh = lambda x: [x[r * nl:(r + 1) * nl] for r in range(p)]
        out, state = O.ulysses_forward(sh(q), sh(k), sh(v), kind)
        dq, dk, dv = O.ulysses_backward(sh(do), state, kind)
        cat = lambda xs: np.concatenate(xs, 0)
        # bitwise: same fixed-order arithmetic as the reference
        assert np.array_equal(cat(out), g[f"case{ci}_o"])
        assert np.array_equal(cat(dq), g[f"case{ci}_dq"])
        assert np.array_equal(cat(dk), g[f"case{ci}_dk"])
        assert np.array_equal(cat(dv), g[f"case{ci}_dv"])
        # ledger: 8 a2a of aggregate n*b*d, egress (nbd/P)(P-1)/P each (test_ulysses.py:220-222)
        led = g[f"case{ci}_ledger"]
        assert len(led) == 8
        assert all(int(a) == n * b * h * hd for a, _ in led)
        assert all(int(e) == O.all_to_all_metering(nl * b * h * hd, p)[1] for _, e in led)

    def test_gqa_reduces_to_mha(self):
        g = load("attn_small.npz")
        ci = 1
        p, n, b, h, hd, causal, seed = (int(x) for x in g[f"case{ci}_meta"])
        q, k, v, do = (g[f"case{ci}_{t}"].astype(np.float64) for t in ("q", "k", "v", "do"))
        c, _ = O.local_attention(q, k, v, "causal")
        # GQA with kv replicated per group equals MHA on the replicated tensors
        kg, vg = k[:, :, ::2], v[:, :, ::2]
        c_gqa, _ = O.local_attention(q, kg, vg, "causal")
        c_rep, _ = O.local_attention(q, np.repeat(kg, 2, axis=2), np.repeat(vg, 2, axis=2), "causal")
        assert np.array_equal(c_gqa, c_rep)
        _, dk_g, dv_g = O.local_attention_backward(q, kg, vg, do, "causal")
        _, dk_r, dv_r = O.local_attention_backward(q, np.repeat(kg, 2, axis=2),
                                                   np.repeat(vg, 2, axis=2), do, "causal")
        np.testing.assert_allclose(dk_g, dk_r[:, :, 0::2] + dk_r[:, :, 1::2], rtol=0, atol=1e-14)
        np.testing.assert_allclose(dv_g, dv_r[:, :, 0::2] + dv_r[:, :, 1::2], rtol=0, atol=1e-14)
        assert np.array_equal(c, O.local_attention(q, k, v, "causal")[0])


@pytest.mark.slow
class TestConfig1Golden:
    def test_config1_forward_backward(self):
        g = load("config1.npz")
        p, n, b, h, hd, seed = (int(x) for x in g["meta"])
        rows = g["rows"]
        q, k, v, do = (O.make_tensor((n, b, h, hd), seed, s) for s in (1, 2, 3, 4))
        import hashlib
        hsh = hashlib.sha256()
        for a in (q, k, v, do):
            hsh.update(np.ascontiguousarray(a).tobytes())
        assert hsh.hexdigest()[:16] == bytes(g["inputs_digest"]).decode()
        nl = n // p
        sh = lambda x: [x[r * nl:(r + 1) * nl] for r in range(p)]
        for kind in ("none", "causal"):
            out, state = O.ulysses_forward(sh(q), sh(k), sh(v), kind)
            o = np.concatenate(out, 0)
            assert np.array_equal(o[rows], g[f"{kind}_o_rows"])
            if kind == "causal":
                dq, dk, dv = (np.concatenate(x, 0) for x in O.ulysses_backward(sh(do), state, kind))
                assert np.array_equal(dq[rows], g["causal_dq_rows"])
                assert np.array_equal(dk[rows], g["causal_dk_rows"])
                assert np.array_equal(dv[rows], g["causal_dv_rows"])
