"""NEXT-N1 on the GPU: the Eq. 11 front end (token matrices -> prompt vectors) vs the
oracle (oracle.prompt_vector, fp64, pinned to the literal Gram-matrix Eq. 11), and the
whole path from token matrices vs the literal SCS of PAPER.md Eq. 11."""
import numpy as np
import pytest

import gen
import oracle
from parity import compare

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("remoe_lib_built")]
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_18674_b200 as remoe  # noqa: E402


def _embed(tok, off, want_f32=True):
    t = torch.from_numpy(tok.view(np.int16)).cuda()
    o = torch.from_numpy(off).cuda()
    ob, of = remoe.embed(t, o, want_f32=want_f32)
    torch.cuda.synchronize()
    return ob.cpu().numpy().view(np.uint16), (of.cpu().numpy() if of is not None else None)


@pytest.mark.parametrize("dim", [8, 40, 384, 1024, 4096])
def test_embed_matches_oracle(dim):
    tok, off, _ = gen.token_prompts(7 + dim, 37, dim, min_len=0, max_len=300, zero_token_every=11)
    ob, of = _embed(tok, off)
    x = gen.bf16_bits_to_f32(tok).astype(np.float64)
    for p in range(37):
        rows = x[off[p]:off[p + 1]]
        rows = rows[(rows * rows).sum(1) > 0]          # zero tokens contribute nothing (R17)
        ref = oracle.prompt_vector(rows) if len(rows) else np.zeros(dim)
        n = max(1, len(rows))
        np.testing.assert_allclose(of[p], ref, rtol=0, atol=n * 2e-6)
    # the bf16 output is the round-to-nearest-even of the fp32 output
    np.testing.assert_array_equal(ob, gen.f32_to_bf16_bits(of))
    empty = np.nonzero(off[1:] == off[:-1])[0]
    assert np.all(of[empty] == 0)


def test_embed_is_batch_position_invariant():
    tok, off, _ = gen.token_prompts(3, 20, 256, max_len=90)
    _, of = _embed(tok, off)
    # the same prompts, reversed: identical vectors bit for bit
    order = np.arange(19, -1, -1)
    lens = off[1:] - off[:-1]
    tok2 = np.concatenate([tok[off[p]:off[p + 1]] for p in order])
    off2 = np.zeros(21, np.int64)
    off2[1:] = np.cumsum(lens[order])
    _, of2 = _embed(tok2, off2)
    np.testing.assert_array_equal(of2, of[order])


def test_token_prompts_end_to_end_vs_literal_eq11():
    """History and queries given as token matrices: embed -> build -> query.  Scores vs the
    literal Eq. 11 (oracle.scs_gram on the token matrices): within the bf16 rounding of the
    stored prompt vectors (|d| <= 5e-3); exact parity vs the oracle on those bf16 vectors;
    a query that repeats a history prompt retrieves it first."""
    D, P, Q, k = 384, 300, 12, 5
    tok, off, _ = gen.token_prompts(11, P + Q, D, min_len=4, max_len=40, n_topics=6)
    ob, _ = _embed(tok, off, want_f32=False)
    hist, qv = ob[:P].copy(), ob[P:].copy()
    qv[0] = hist[17]                                      # a repeated prompt
    act = gen.store_act(5, P, 4, 8, 2)
    sps = remoe.Sps(hist, act, max_k=8)
    ids, sc, pred = sps.query(torch.from_numpy(qv.view(np.int16)).cuda(), k)
    ids, sc, pred = ids.cpu().numpy(), sc.cpu().numpy(), pred.cpu().numpy()
    assert compare(qv, hist, act, k, ids, sc, pred).ok()
    assert ids[0, 0] == 17
    x = gen.bf16_bits_to_f32(tok).astype(np.float64)
    for i in range(1, Q):
        qt = x[off[P + i]:off[P + i + 1]]
        lit = np.array([oracle.scs_gram(qt, x[off[j]:off[j + 1]]) for j in range(P)])
        assert np.abs(sc[i] - lit[ids[i]]).max() <= 5e-3
        best = np.sort(lit)[::-1][:k]
        assert np.abs(np.sort(sc[i])[::-1] - best).max() <= 5e-3
