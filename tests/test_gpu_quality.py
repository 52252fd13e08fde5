"""NEXT-N4 on the GPU: the JS-divergence kernel vs the oracle (pinned to scipy and the
closed forms in test_oracle_pins), and the quality ordering of the paper's predictors
(P:675): SPS (exact BF top-alpha) below DOP (historical mean) below EF (uniform)."""
import os
import sys

import numpy as np
import pytest

import gen
import oracle

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("remoe_lib_built")]
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_18674_b200 as remoe  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))


def test_js_kernel_matches_oracle():
    rng = np.random.default_rng(1)
    for B, L, E in [(3, 1, 2), (17, 27, 64), (5, 32, 8), (4, 3, 256)]:
        p = rng.random((B, L, E)).astype(np.float32)
        p[rng.random((B, L, E)) < 0.3] = 0
        p[..., 0] += 1e-3
        p /= p.sum(-1, keepdims=True)
        q = rng.random((B, L, E)).astype(np.float32)
        q /= q.sum(-1, keepdims=True)
        out = remoe.js_divergence(torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()).cpu().numpy()
        ref = np.array([oracle.js_divergence(p[b], q[b]) for b in range(B)])
        np.testing.assert_allclose(out, ref, rtol=0, atol=2e-6)
    # closed forms through the kernel: identical -> 0, disjoint -> 1, [.5,.5] vs [.9,.1]
    P = torch.tensor([[[0.5, 0.5]], [[1.0, 0.0]], [[0.5, 0.5]]], device="cuda")
    Q = torch.tensor([[[0.5, 0.5]], [[0.0, 1.0]], [[0.9, 0.1]]], device="cuda")
    out = remoe.js_divergence(P, Q).cpu().numpy()
    np.testing.assert_allclose(out, [0.0, 1.0, 0.146793], atol=2e-6)
    # many layers: the per-layer values need > 48 KB of shared memory (L = 20,000 x 4 B)
    L = 20_000
    p = np.full((2, L, 2), 0.5, np.float32)
    q = np.zeros((2, L, 2), np.float32)
    q[0, :, 0] = 1.0          # [.5,.5] vs [1,0] on every layer
    q[1] = 0.5                # identical
    out = remoe.js_divergence(torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()).cpu().numpy()
    ref = oracle.js_divergence(p[0, :1], q[0, :1])
    np.testing.assert_allclose(out, [ref, 0.0], atol=1e-4)  # fp32 sum of 20,000 layer values


def test_sps_beats_dop_beats_ef():
    import quality
    res, pred, truth = quality.evaluate("c2", n=20_000, held_out=128, k=15)
    assert res["SPS"] < res["DOP"] < res["EF"], res
    # NEXT-N2: the clustering tree predicts far better than DOP with a fraction of the
    # Eq. 11 evaluations of BF ("more than 10 times faster than BF")
    assert res["TREE"] < res["DOP"], res
    assert res["tree"]["mean_evals"] * 10 < res["tree"]["evals_bf"], res
    # the harness's JS numbers agree with the oracle on a sample
    for i in range(0, 128, 31):
        ref = oracle.js_divergence(pred[i], truth[i])
        js = remoe.js_divergence(torch.from_numpy(pred[i:i + 1]).cuda(),
                                 torch.from_numpy(truth[i:i + 1]).cuda()).item()
        assert abs(js - ref) <= 2e-6
