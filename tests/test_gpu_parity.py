"""GPU (libakv, sm_100a) vs CPU oracle parity — SURVEY §8(c).

Bit-exact: stored planes, ColMax/RowMax, K tier masks, V tier masks (with
the D11 knife-edge protocol, plus an injection check that must be 100 %
exact), selection sets, AccessCounter totals.  Within 1e-3 (per vector,
|gpu-ref| <= 1e-3|ref| + 1e-3 max|ref|): scores and outputs.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import attention_decode as OA
from oracle import half_bits as ohb
from oracle.align_core import AlignConfig as OAlignConfig
from oracle.analysis import relative_error_histogram
from oracle.kv_store import PlaneTensor as OPlane
from paper_2409_16546_b200 import AlignConfig, DegenerateInputError, KVStore
from paper_2409_16546_b200 import attention_decode as AD
from paper_2409_16546_b200.synth import generate_batch
from tests.gpu_helpers import Case, check_head, close


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("n", [1, 7, 255, 256, 257, 600])
def test_planes_and_sidecars_bitexact(n):
    c = Case(B=2, Hkv=3, n=n, seed=100 + n)
    for which, src in (("k", c.K), ("v", c.V)):
        p0, p1, p2 = c.store.export_planes(which)
        for u in range(6):
            b, h = divmod(u, 3)
            ref = OPlane.from_words(src[u])
            assert np.array_equal(p0[b, h], ref.plane0)
            assert np.array_equal(p1[b, h], ref.plane1)
            assert np.array_equal(p2[b, h], ref.plane2)
    cm = c.store.colmax().cpu().numpy()
    rm = c.store.rowmax().cpu().numpy().view(np.uint16)
    for u in range(6):
        b, h = divmod(u, 3)
        o = c.ostore(u)
        assert np.array_equal(cm[b, h].astype(np.uint16), o.colmax)
        assert np.array_equal(rm[b, h, :n], o.rowmax)
    assert (c.store.lengths == n).all()


def test_append_rejects_nonfinite_with_position():
    st = KVStore(1, 2, 128, 512)
    k = torch.randn(1, 2, 5, 128).half()
    v = torch.randn(1, 2, 5, 128).half()
    st.append(k, v)
    k2 = torch.randn(1, 2, 128).half()
    v2 = torch.randn(1, 2, 128).half()
    v2[0, 1, 77] = float("inf")
    with pytest.raises(ValueError, match=r"non-finite half word 0x7C00 in V at batch 0, kv-head 1, token 5, channel 77"):
        st.append_token(k2, v2)
    # per-unit semantics (each unit is one SPEC store): the finite unit commits, the offender does not
    assert st.lengths.tolist() == [[6, 5]]
    assert st.lengths_dev.cpu().tolist() == [6, 5]
    st.rewind(5)
    kb = torch.randn(1, 2, 3, 128).half()
    kb[0, 0, 2, 9] = float("nan")
    with pytest.raises(ValueError, match=r"in K at batch 0, kv-head 0, token 7, channel 9"):
        st.append(kb, torch.randn(1, 2, 3, 128).half())
    assert st.lengths.tolist() == [[5, 8]]  # unit (0,1) committed its 3 finite tokens
    st.rewind(5)
    st.append_token(k2, torch.randn(1, 2, 128).half())
    assert st.lengths.tolist() == [[6, 6]]


def _compare_case(c: Case, cfg=AlignConfig(), ocfg=OAlignConfig(), strategy="element", force=None,
                  max_edge_frac=0.1):
    """Every q-head against the oracle through oracle.parity.check_head.  D11 knife-edge
    heads skip only the selection / V-mask / V-counter asserts on the affected rows and
    columns; the injection check runs for every head.  The knife-edge count is returned and
    bounded (the synthetic cases produce almost none)."""
    r = c.gpu(cfg=cfg, strategy=strategy, force_tier=force)
    s = r.scores.cpu().numpy()
    p = r.probs.cpu().numpy()
    o = r.o.cpu().numpy()
    kt = r.k_tiers.cpu().numpy()
    vt = r.v_tiers.cpu().numpy()
    cnt = r.counters.cpu().numpy()
    tg = r.targets.cpu().numpy()
    edges = heads = 0
    for u, b, hq, j in c.units():
        ref = c.oracle(u, j, ocfg, strategy=strategy, force_tier=force)
        fail, edge = check_head(ref, k_tiers=kt[b, hq], o=o[b, hq], counters=cnt[b, hq], sel=r.selection(b, hq),
                                v_tiers=vt[b, hq], s=s[b, hq], p=p[b, hq], targets=tg[b, hq],
                                v_head=c.V[u] >> 8, cfg=ocfg, strategy=strategy, force=force)
        assert not fail, (u, j, fail)
        edges += edge
        heads += 1
    assert edges <= max(1, int(max_edge_frac * heads)), f"{edges} knife-edge heads of {heads}"
    r.knife_edges = edges
    return r


@pytest.mark.parametrize("n", [16, 256, 1000])
def test_mha_parity(n):
    _compare_case(Case(B=2, Hkv=2, g=1, n=n, seed=n))


@pytest.mark.parametrize("g", [2, 4, 8])
def test_gqa_parity(g):
    _compare_case(Case(B=1, Hkv=2, g=g, n=513, seed=40 + g))


@pytest.mark.parametrize("g", [2, 8])
def test_flat_scales_parity(g):
    """Paper-like regime (U[-0.5,0.5]): many T12/T16 reads and element-path V rows
    (g = 8: chunks mixing all three K tier variants in the tensor-core qk)."""
    c = Case(B=2, Hkv=2, g=g, n=700, seed=5, lo=-0.5, hi=0.5)
    r = _compare_case(c)
    st = r.v_stats()
    assert st.t12 + st.t16 > st.elements_read * 0.001


@pytest.mark.parametrize("margin,zero_skip,g", [(-2, True, 2), (4, True, 2), (0, False, 2), (0, True, 4),
                                               (3, False, 4)])
def test_config_parity(margin, zero_skip, g):
    c = Case(B=1, Hkv=2, g=g, n=300, seed=77)
    c.Q[0, 0, :5] = 0  # zero q channels exercise D1
    c.Q[1, :, 40:48] = 0  # ... in every head of a unit: SKIP for the whole group under zero_skip
    c.q = torch.from_numpy(c.Q.view(np.int16)).view(c.B, c.Hkv * c.g, 128)
    _compare_case(c, AlignConfig(margin, zero_skip), OAlignConfig(margin, zero_skip))


def test_row_strategy_parity():
    _compare_case(Case(B=1, Hkv=2, g=2, n=400, seed=9, lo=-1, hi=1), strategy="row")


@pytest.mark.parametrize("tier,g", [(8, 1), (12, 1), (16, 1), (8, 4), (12, 4), (16, 8)])
def test_forced_tier_parity(tier, g):
    _compare_case(Case(B=1, Hkv=2, g=g, n=300, seed=3), force=tier)


def test_forced_t16_equals_reference_paths():
    """SPEC.md:584 on the GPU: forced T16 == reference_scores/reference_output (bit-identical)."""
    c = Case(B=2, Hkv=2, g=2, n=333, seed=21)
    r = c.gpu(force_tier=16)
    s_ref = AD.reference_scores(c.q, c.store)
    assert torch.equal(r.scores, s_ref)
    o_ref = AD.reference_output(r.probs, c.store)
    assert torch.equal(r.o, o_ref)
    # ... and agrees with a plain torch fp32 attention over the stored fp16 words
    K = torch.from_numpy(c.K.view(np.int16)).view(torch.float16).float().cuda()
    V = torch.from_numpy(c.V.view(np.int16)).view(torch.float16).float().cuda()
    q = c.q.cuda().view(torch.float16).float().view(4, 2, 128)
    s_t = torch.einsum("ugd,und->ugn", q, K) / np.sqrt(128)
    p_t = torch.softmax(s_t.double(), -1).float()
    o_t = torch.einsum("ugn,und->ugd", p_t, V)
    assert close(r.o.view(4, 2, 128).cpu().numpy(), o_t.cpu().numpy())


@pytest.mark.parametrize("g", [1, 4])
def test_baseline_truncated_parity(g):
    c = Case(B=1, Hkv=2, g=g, n=300, seed=8)
    r = c.gpu()
    s_b, o_b = AD.baseline_truncated(c.q, c.store, r.probs, 13)
    for u, b, hq, j in c.units():
        s_ref, o_ref = OA.baseline_truncated(c.Q[u, j], c.K[u], r.probs[b, hq].cpu().numpy().astype(np.float64),
                                             c.V[u], 13)
        assert close(s_b[b, hq].cpu().numpy(), s_ref)
        assert close(o_b[b, hq].cpu().numpy(), o_ref)


def test_stepwise_api_matches_fused_step():
    c = Case(B=1, Hkv=2, g=2, n=500, seed=31)
    fused = c.gpu()
    sv = AD.scores_aligned(c.q, c.store)
    assert torch.equal(sv.s, fused.scores)
    assert torch.equal(sv.k_tiers, fused.k_tiers)
    p = AD.softmax(sv)
    assert torch.equal(p.p, fused.probs)
    est = AD.estimate_output(p, c.store)
    assert torch.equal(est.o_est, fused.o_est)
    o, vstats, vt = AD.output_aligned(p, c.store, est, export_v_tiers=True)
    assert torch.equal(o, fused.o)
    assert torch.equal(vt, fused.v_tiers)
    with pytest.raises(ValueError, match="missing o_est"):
        AD.output_aligned(p, c.store, None)


def test_degenerate_q_raises():
    c = Case(B=1, Hkv=1, g=1, n=20, seed=2)
    with pytest.raises(DegenerateInputError, match="degenerate dot product"):
        AD.decode_step(torch.zeros(1, 1, 128, dtype=torch.float16), c.store)


def test_spec_examples_embedded():
    """SPEC.md:321 (d=2 example embedded in d=128 with zero channels)."""
    st = KVStore(1, 1, 128, 256)
    k = np.zeros(128, np.uint16)
    k[0], k[1] = ohb.encode(1.0), ohb.encode(7.0)
    st.append_token(torch.from_numpy(k.view(np.int16)), torch.zeros(128, dtype=torch.int16))
    q = np.zeros(128, np.uint16)
    q[0] = ohb.encode(1.0)
    sv = AD.scores_aligned(torch.from_numpy(q.view(np.int16)), st)
    assert sv.s.item() == pytest.approx(1.0 / np.sqrt(128), rel=1e-7)  # d=128 scaling
    assert sv.k_tiers[0, 0, 0].item() == 16 and (sv.k_tiers[0, 0, 1:] == 0).all()
    assert sv.k_stats.bits_read == 16
    # one-hot p -> o = V row exactly
    st2 = KVStore(1, 1, 128, 256)
    K = np.zeros((3, 128), np.uint16)
    K[:, 0] = ohb.encode_array([1.0, 2000.0, 1.0])
    V = ohb.encode_array(np.random.default_rng(0).standard_normal((3, 128)))
    st2.append(torch.from_numpy(K.view(np.int16)), torch.from_numpy(V.view(np.int16)))
    r = AD.decode_step(torch.from_numpy(q.view(np.int16)), st2)
    assert np.array_equal(r.o[0, 0].cpu().numpy(), ohb.decode_array(V[1]).astype(np.float32))
    # ... and through the GQA kernels (4 q-heads on the kv-head)
    q4 = np.tile(q, (4, 1)).reshape(1, 4, 128)
    r4 = AD.decode_step(torch.from_numpy(q4.view(np.int16)), st2)
    for j in range(4):
        assert np.array_equal(r4.o[0, j].cpu().numpy(), ohb.decode_array(V[1]).astype(np.float32))


def test_error_histograms_match_oracle():
    """Aligned-vs-full-fp16 error histograms (A-hist) within +-1 pp of the oracle's."""
    c = Case(B=2, Hkv=2, g=1, n=1024, seed=7)
    r = c.gpu()
    rr = c.gpu(force_tier=16)
    o_ref_gpu = AD.reference_output(r.probs, c.store)
    rnd = ohb.float16_round
    gq, oq, gs, os_ = [], [], [], []
    for u, b, hq, j in c.units():
        ref = c.oracle(u, j)
        s_ref = OA.reference_scores(c.Q[u, j], c.K[u])
        o_ref = OA.reference_output(ref.p, c.V[u])
        gq.append(relative_error_histogram(rnd(r.scores[b, hq].cpu().numpy()), rnd(rr.scores[b, hq].cpu().numpy())))
        oq.append(relative_error_histogram(rnd(ref.s), rnd(s_ref)))
        gs.append(relative_error_histogram(rnd(r.o[b, hq].cpu().numpy()), rnd(o_ref_gpu[b, hq].cpu().numpy())))
        os_.append(relative_error_histogram(rnd(ref.o), rnd(o_ref)))
    assert np.abs(np.mean(gq, 0) - np.mean(oq, 0)).max() <= 0.01
    assert np.abs(np.mean(gs, 0) - np.mean(os_, 0)).max() <= 0.01


def test_determinism_and_ragged_lengths():
    c = Case(B=2, Hkv=2, g=2, n=700, seed=13)
    a = c.gpu()
    b = c.gpu()
    assert torch.equal(a.o, b.o) and torch.equal(a.counters, b.counters)
    # ragged: shorten unit (b=0, h=1) on device -> its output equals the oracle on its first 300 tokens
    c.store.lengths_dev[1] = 300
    c.store._host_len[1] = 300
    r = c.gpu()
    from oracle.kv_store import KVStore as OStore
    st = OStore(128)
    st.append_rows(c.K[1][:300], c.V[1][:300])
    st.colmax = c.store.colmax()[0, 1].cpu().numpy().astype(np.uint16)  # running max is not rewound
    for j in range(2):
        ref = OA.decode_head(c.Q[1, j], st)
        assert np.array_equal(r.k_tiers[0, 2 + j].cpu().numpy(), ref.k_tiers)
        assert close(r.o[0, 2 + j].cpu().numpy(), ref.o)
    # the untouched units are unchanged
    assert torch.equal(r.o[0, :2], a.o[0, :2]) and torch.equal(r.o[1], a.o[1])


def test_decode_graph_matches_decode_step():
    """DecodeGraph (CUDA graph of append + decode) == eager append_token + decode_step."""
    B, Hkv, g, n = 2, 2, 2, 500
    K, V, Q = generate_batch(B, Hkv, n, 128, g, 5)
    d = 128
    kt = torch.from_numpy(K.view(np.int16)).view(B, Hkv, n, d)
    vt = torch.from_numpy(V.view(np.int16)).view(B, Hkv, n, d)
    q = torch.from_numpy(Q.view(np.int16)).view(B, Hkv * g, d)
    a = KVStore(B, Hkv, d, 512)
    a.append(kt[:, :, : n - 1], vt[:, :, : n - 1])
    a.append_token(kt[:, :, n - 1], vt[:, :, n - 1])
    ref = AD.decode_step(q, a)
    b = KVStore(B, Hkv, d, 512)
    b.append(kt[:, :, : n - 1], vt[:, :, : n - 1])
    dg = AD.DecodeGraph(b, g, rewind_to=n - 1).capture()
    for _ in range(3):  # replays are idempotent with rewind_to
        out = dg.step(q, kt[:, :, n - 1], vt[:, :, n - 1])
    dg.check()
    assert torch.equal(out, ref.o.cpu())
    # in-place host buffers (the serving form): fill, replay, read
    dg.host_q.copy_(q)
    out2 = dg.step()
    assert torch.equal(out2, ref.o.cpu())


def test_many_units_items_span_warps_and_units():
    """B=16 x 32 kv-heads x 4 pages = 2048 (unit, page) items, more than resident warps:
    warps cross unit boundaries (Rule-1 re-evaluation, page-table rows, TMA ring cursors)."""
    c = Case(B=16, Hkv=32, g=1, n=1024, seed=77)
    r = c.gpu()
    kt = r.k_tiers.cpu().numpy()
    o = r.o.cpu().numpy()
    for u, b, hq, j in c.units():
        if u % 8:  # oracle on every 8th unit keeps the CPU side to seconds
            continue
        ref = c.oracle(u, j)
        assert np.array_equal(kt[b, hq], ref.k_tiers), u
        assert close(o[b, hq], ref.o), u


def test_gqa_many_pages():
    """GQA g=4 over 6 pages per unit (two q-head passes are not needed: g <= 4)."""
    _compare_case(Case(B=2, Hkv=4, g=4, n=1500, seed=91))


@pytest.mark.parametrize("zin,zout", [(False, False), (True, False), (False, True)])
def test_decode_graph_copy_modes(zin, zout):
    B, Hkv, g, n = 2, 2, 1, 300
    K, V, Q = generate_batch(B, Hkv, n, 128, g, 6)
    d = 128
    kt = torch.from_numpy(K.view(np.int16)).view(B, Hkv, n, d)
    vt = torch.from_numpy(V.view(np.int16)).view(B, Hkv, n, d)
    q = torch.from_numpy(Q.view(np.int16)).view(B, Hkv * g, d)
    a = KVStore(B, Hkv, d, 512)
    a.append(kt, vt)
    ref = AD.decode_step(q, a)
    b = KVStore(B, Hkv, d, 512)
    b.append(kt[:, :, : n - 1], vt[:, :, : n - 1])
    dg = AD.DecodeGraph(b, g, rewind_to=n - 1, zero_copy_in=zin, zero_copy_out=zout).capture()
    out = dg.step(q, kt[:, :, n - 1], vt[:, :, n - 1])
    assert torch.equal(out, ref.o.cpu())


def test_long_context_beyond_register_page_table():
    """n = 33000 tokens = 129 pages: pages >= 128 take the page-table fallback path."""
    _compare_case(Case(B=1, Hkv=1, g=1, n=33000, seed=123))


def test_gqa_long_context():
    """g = 8 over 40 pages (n > 8192: the 1024-thread select; qk5 rings continuous across
    many pages of a unit; pv quad path)."""
    _compare_case(Case(B=1, Hkv=1, g=8, n=10000, seed=17))


@pytest.mark.parametrize("g,n,lo,hi", [(1, 1500, -4.0, 4.0), (1, 1100, -0.5, 0.5), (2, 700, -0.5, 0.5),
                                       (4, 1500, -4.0, 4.0), (4, 700, -0.5, 0.5), (8, 600, -4.0, 4.0)])
def test_fast_path_parity(g, n, lo, hi):
    """The serving path (no v-tier export: pv6 T8 stages on the tensor cores, plan rows through
    the SIMD rule, and at paper-like scales (-0.5, 0.5) the DENSE stages for g <= 2) against
    the oracle, with V-side counters equal to the export run's."""
    c = Case(B=2, Hkv=2, g=g, n=n, seed=60 + g, lo=lo, hi=hi)
    r = AD.decode_step(c.q, c.store)
    o = r.o.cpu().numpy()
    cnt = r.counters.cpu().numpy()
    ref_e = c.gpu()  # export run: exact V-side counters for comparison
    cnt_e = ref_e.counters.cpu().numpy()
    for u, b, hq, j in c.units():
        ref = c.oracle(u, j)
        assert close(o[b, hq], ref.o), (g, u, j)
    assert np.array_equal(cnt, cnt_e)  # same tier decisions -> same element counts


def test_decode_graph_gqa_matches_eager():
    """DecodeGraph (CUDA graph: append + qk5 + select + pv quad path + combine) with g = 4
    equals the eager step bit for bit."""
    B, Hkv, g, n, d = 1, 2, 4, 700, 128
    K, V, Q = generate_batch(B, Hkv, n, d, g, 12)
    kt = torch.from_numpy(K.view(np.int16)).view(B, Hkv, n, d)
    vt = torch.from_numpy(V.view(np.int16)).view(B, Hkv, n, d)
    q = torch.from_numpy(Q.view(np.int16)).view(B, Hkv * g, d)
    a = KVStore(B, Hkv, d, 1024)
    a.append(kt, vt)
    ref = AD.decode_step(q, a)
    b = KVStore(B, Hkv, d, 1024)
    b.append(kt[:, :, : n - 1], vt[:, :, : n - 1])
    dg = AD.DecodeGraph(b, g, rewind_to=n - 1).capture()
    for _ in range(2):  # replays rewind and re-append the same token
        out = dg.step(q, kt[:, :, n - 1], vt[:, :, n - 1])
        assert torch.equal(out, ref.o.cpu().view_as(out))


def _zero_v_channel_and_underflow(K, V, Q):
    """Unit 0: V channels 5 and 77 all zero (o_est_r == 0 -> unknown Rule-2 target), and
    one token whose score underflows p to exactly 0 (fp32 and float64) for every q-head of
    the unit: q made non-negative, that token's K row = -60000."""
    V[0][:, [5, 77]] = 0
    Q[0] = Q[0] & 0x7FFF
    K[0][3] = np.float16(-60000.0).view(np.uint16)
    # unit 1: a zero V channel only
    V[1][:, 0] = 0


@pytest.mark.parametrize("g", [1, 2, 4])
def test_unknown_target_overrides_p_zero(g):
    """a dim with o_est_r == 0 forces T16 on every read contributing to it,
    including rows whose p_t underflowed to 0 (the kernels used to read those rows at T8).
    V masks, V counters and the injection check must match the oracle."""
    c = Case(B=1, Hkv=2, g=g, n=300, seed=4, mutate=_zero_v_channel_and_underflow)
    r = _compare_case(c)
    vt = r.v_tiers.cpu().numpy()
    p = r.probs.cpu().numpy()
    for j in range(g):
        assert p[0, j, 3] == 0.0  # the underflow row is exactly 0 ...
        sel = set(r.selection(0, j).tolist())
        rows = [t for t in range(c.n) if t not in sel]
        assert (vt[0, j][rows][:, [5, 77]] == 16).all()  # ... and still read at T16 on the unknown dims
        assert vt[0, j, 3, 5] == 16 and vt[0, j, 3, 77] == 16
    # the serving path (no V-mask export) takes the same decisions: identical counters
    r2 = AD.decode_step(c.q, c.store)
    assert torch.equal(r2.counters, r.counters)
    assert close(r2.o.cpu().numpy(), r.o.cpu().numpy())


def test_decode_graph_errors_are_sticky_and_capacity_guarded():
    """A rejected append inside a replay stays visible after later clean replays (sticky
    device status); check() resyncs the host length mirror; a full store refuses to replay."""
    B, Hkv, g, n = 1, 2, 1, 254
    K, V, Q = generate_batch(B, Hkv, n + 2, 128, g, 3)
    d = 128
    kt = torch.from_numpy(K.view(np.int16)).view(B, Hkv, n + 2, d)
    vt = torch.from_numpy(V.view(np.int16)).view(B, Hkv, n + 2, d)
    q = torch.from_numpy(Q.view(np.int16)).view(B, Hkv * g, d)
    st = KVStore(B, Hkv, d, 256)  # capacity 256
    st.append(kt[:, :, :n], vt[:, :, :n])
    dg = AD.DecodeGraph(st, g).capture()
    bad = kt[:, :, n].clone()
    bad[0, 1, 9] = 0x7C00  # +inf in unit (0, 1)
    dg.step(q, bad, vt[:, :, n])
    dg.step(q, kt[:, :, n + 1], vt[:, :, n + 1])  # a clean replay does not clear the error
    with pytest.raises(ValueError, match=r"non-finite K channel 9\) at batch 0, kv-head 1"):
        dg.check()
    assert st.lengths.tolist() == [[256, 255]]  # unit (0,1) rejected one token
    assert st.lengths_dev.cpu().tolist() == [256, 255]
    with pytest.raises(ValueError, match="store is full"):
        dg.step(q, kt[:, :, n + 1], vt[:, :, n + 1])


@pytest.mark.parametrize("chunks", [(37, 300, 1), (256, 255, 2), (1, 511, 90), (700,)])
def test_prefill_writer_spans_bitexact(chunks):
    """akv_append_ws (page-span tiles): successive bulk appends starting mid-page and mid
    16-token group must leave the planes / sidecars equal to the oracle's (merge path at
    both span ends), and the old bytes of the page outside each span untouched."""
    n = sum(chunks)
    B, Hkv = 1, 3
    K, V, _ = generate_batch(B, Hkv, n, 128, 1, seed=5 + n)
    st = KVStore(B, Hkv, 128, 1024)
    kt = torch.from_numpy(K.view(np.int16)).view(B, Hkv, n, 128)
    vt = torch.from_numpy(V.view(np.int16)).view(B, Hkv, n, 128)
    t = 0
    for c in chunks:
        st.append(kt[:, :, t:t + c], vt[:, :, t:t + c])
        t += c
    st.check()
    for which, src in (("k", K), ("v", V)):
        p0, p1, p2 = st.export_planes(which)
        for u in range(Hkv):
            ref = OPlane.from_words(src[u])
            assert np.array_equal(p0[0, u], ref.plane0)
            assert np.array_equal(p1[0, u], ref.plane1)
            assert np.array_equal(p2[0, u], ref.plane2)
    cm = st.colmax().cpu().numpy()
    rm = st.rowmax().cpu().numpy().view(np.uint16)
    for u in range(Hkv):
        from oracle.kv_store import KVStore as OStore
        o = OStore(128)
        o.append_rows(K[u], V[u])
        assert np.array_equal(cm[0, u].astype(np.uint16), o.colmax)
        assert np.array_equal(rm[0, u, :n], o.rowmax)
    assert (st.lengths == n).all()


def test_prefill_writer_earliest_offender_and_capacity():
    """The fused validation reports the earliest offending word over all page spans (token,
    then K before V, then channel), refuses the unit's whole append (length, ColMax
    unchanged) and commits the other units; an append beyond capacity is refused."""
    st = KVStore(1, 2, 128, 1024)
    st.append(torch.randn(1, 2, 100, 128).half(), torch.randn(1, 2, 100, 128).half())
    cm0 = st.colmax().clone()
    k = torch.randn(1, 2, 600, 128).half()
    v = torch.randn(1, 2, 600, 128).half()
    k[0, 0, 550, 3] = float("inf")   # later span
    v[0, 0, 400, 100] = float("nan")  # earlier token (V): reported
    k[0, 0, 400, 120] = float("-inf")  # same token, K before V: reported first
    k[0, 1, 10] *= 1000  # unit 1 commits (ColMax grows)
    with pytest.raises(ValueError, match=r"in K at batch 0, kv-head 0, token 500, channel 120"):
        st.append(k, v)
    assert st.lengths.tolist() == [[100, 700]]
    cm = st.colmax()
    assert torch.equal(cm[0, 0], cm0[0, 0])
    assert bool((cm[0, 1] >= cm0[0, 1]).all()) and not torch.equal(cm[0, 1], cm0[0, 1])
    st2 = KVStore(1, 1, 128, 256)
    st2.append(torch.randn(1, 1, 200, 128).half(), torch.randn(1, 1, 200, 128).half())
    with pytest.raises(ValueError, match="capacity"):
        st2.append(torch.randn(1, 1, 100, 128).half(), torch.randn(1, 1, 100, 128).half())
    assert st2.lengths.tolist() == [[200]]


def test_metered_reads_match_oracle():
    """KVStore.read_element / read_channel / read_elements on the device (akv_read_elements)
    against the oracle's metered reads: rebuilt words bit-exact at every
    tier (SKIP -> 0, 0 bits), AccessCounter totals equal, K and V, pages crossed."""
    from oracle.kv_store import AccessCounter as OCounter
    from paper_2409_16546_b200 import AccessCounter
    c = Case(B=2, Hkv=2, n=600, seed=77)
    rng = np.random.default_rng(3)
    for which in ("k", "v"):
        units = rng.integers(0, 4, 500)
        toks = rng.integers(0, 600, 500)
        chans = rng.integers(0, 128, 500)
        tiers = rng.choice([0, 8, 12, 16], 500)
        gc = AccessCounter()
        got = c.store.read_elements(units, toks, chans, tiers, which, gc).cpu().numpy().view(np.uint16)
        oc = OCounter()
        for i in range(500):
            o = c.ostore(int(units[i]))
            plane = o.k if which == "k" else o.v
            ref = o.read_element(plane, int(toks[i]), int(chans[i]), int(tiers[i]), oc)
            assert int(got[i]) == int(ref) & 0xFFFF, (which, i)
        assert (gc.t8, gc.t12, gc.t16) == (oc.t8, oc.t12, oc.t16)
        for tier in (0, 8, 12, 16):
            gc, oc = AccessCounter(), OCounter()
            col = c.store.read_channel(1, 0, 77, tier, gc, which)
            o = c.ostore(2)
            ref = o.read_channel(o.k if which == "k" else o.v, 77, tier, oc)
            assert np.array_equal(col, np.asarray(ref, dtype=np.uint16))
            assert gc.bits_read == oc.bits_read
        gc = AccessCounter()
        assert c.store.read_element(0, 1, 599, 127, 12, gc, which) == \
            c.ostore(1).read_element(c.ostore(1).k if which == "k" else c.ostore(1).v, 599, 127, 12, OCounter())
    with pytest.raises(IndexError):
        c.store.read_element(0, 0, 600, 0, 8, AccessCounter())


def test_append_at_truncates_and_appends():
    """akv_append_at (include/akv.h): truncate to pos and append there; pos beyond the length
    is rejected with AKV_STATUS_POSITION and leaves the unit unchanged."""
    import ctypes

    from paper_2409_16546_b200 import _lib

    c = Case(B=1, Hkv=2, n=300, seed=31)
    st, L = c.store, _lib.lib()
    K2, V2, _ = generate_batch(1, 2, 1, 128, 1, 77)
    k = torch.from_numpy(K2.view(np.int16)).view(1, 2, 128).cuda()
    v = torch.from_numpy(V2.view(np.int16)).view(1, 2, 128).cuda()
    st.status_dev.zero_()
    _lib.check(L.akv_append_at(ctypes.byref(st.c_store), k.data_ptr(), v.data_ptr(), 297, st.status_dev.data_ptr(),
                               torch.cuda.current_stream().cuda_stream), "akv_append_at")
    torch.cuda.synchronize()
    assert (st.lengths_dev.cpu() == 298).all() and not st.status_dev.cpu().any()
    st._host_len[:] = 298
    cm_before = c.store.colmax().cpu().numpy()
    for which, src, new in (("k", c.K, K2), ("v", c.V, V2)):
        p0, p1, p2 = st.export_planes(which)
        for u in range(2):
            words = np.concatenate([src[u][:297], new[u][:1]])
            ref = OPlane.from_words(words)
            assert np.array_equal(p0[0, u][:298], ref.plane0)
            assert np.array_equal(p1[0, u][:298], ref.plane1)
            assert np.array_equal(p2[0, u][:298], ref.plane2)
    # ColMax is the running max over every appended token (the truncated ones included)
    for u in range(2):
        o = c.ostore(u)
        want = np.maximum(o.colmax, (K2[u][0] & 0x7FFF).astype(np.uint16))
        assert np.array_equal(cm_before[0, u].astype(np.uint16), want)
    # beyond the length: rejected, unchanged
    st.status_dev.zero_()
    _lib.check(L.akv_append_at(ctypes.byref(st.c_store), k.data_ptr(), v.data_ptr(), 299, st.status_dev.data_ptr(),
                               torch.cuda.current_stream().cuda_stream), "akv_append_at")
    torch.cuda.synchronize()
    s = st.status_dev.cpu().numpy()
    assert all((int(w) >> 60) == _lib.STATUS_POSITION for w in s)
    assert (st.lengths_dev.cpu() == 298).all()


def test_append_token_at_api_matches_fresh_store():
    """KVStore.append_token_at: truncate to pos and append through the Python API (the planes
    hold the first pos tokens plus the new one); a position beyond the length is rejected."""
    c = Case(B=1, Hkv=2, n=300, seed=41)
    K2, V2, _ = generate_batch(1, 2, 1, 128, 1, 42)
    k = torch.from_numpy(K2.view(np.int16)).view(1, 2, 128)
    v = torch.from_numpy(V2.view(np.int16)).view(1, 2, 128)
    c.store.append_token_at(250, k, v)
    assert (c.store.lengths == 251).all()
    p0, _, _ = c.store.export_planes("k")
    for u in range(2):
        ref = OPlane.from_words(np.concatenate([c.K[u][:250], K2[u][:1]]))
        assert np.array_equal(p0[0, u][:251], ref.plane0)
    with pytest.raises(ValueError):
        c.store.append_token_at(300, k, v)
