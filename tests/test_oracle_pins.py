"""Pins of the CPU oracle against things other than itself (CPU only, -m "not gpu").

Each test names what fixes the expected value: a value the paper prints
(tests/golden/paper_values.json), a closed form, an invariant, a special case
that reduces to a textbook routine, an error bound, or brute force on tiny
inputs.  DESIGN.md §2 lists the readings R1-R7 these follow.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _rng(seed):
    return np.random.default_rng(seed)


# ---------------------------------------------------------------- fp16 input path
def test_half_to_float_exhaustive(orc):
    """binary16 -> binary32 conversion == numpy's (independent IEEE implementation), all 65536."""
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = h.view(np.float16).astype(np.float32)
    L = orc.lib()
    got = np.array([L.or_half_to_float(int(x)) for x in h], dtype=np.float32)
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin].view(np.uint32), ref[fin].view(np.uint32))
    assert np.all(np.isnan(got[~fin]) == np.isnan(ref[~fin]))


# ---------------------------------------------------------------- R1 encode
def test_encode_spec_worked_example(orc):
    """d=4, g=2, centroids {(0,0),(1,1)}, key (0.9,1.1,0.1,-0.1) -> (1,0)."""
    C = np.array([[[0, 0], [1, 1]], [[0, 0], [1, 1]]], np.float32)
    k = np.array([[0.9, 1.1, 0.1, -0.1]], np.float16)
    assert orc.encode(k, C, 2).tolist() == [[1, 0]]


def test_encode_tie_lowest_index(orc):
    """equidistant to centroids 0 and 1 -> 0 (ties to the lowest index)."""
    C = np.array([[[-1.0], [1.0], [1.0]]], np.float32)
    k = np.array([[0.0]], np.float16)
    assert orc.encode(k, C, 1).tolist() == [[0]]
    C2 = np.array([[[5.0], [1.0], [1.0]]], np.float32)
    assert orc.encode(np.array([[1.0]], np.float16), C2, 1).tolist() == [[1]]


@pytest.mark.parametrize("d,g,c,cbg", [(16, 4, 64, 4), (16, 8, 33, 1), (128, 32, 256, 32), (8, 1, 50, 1)])
def test_encode_brute_force_optimal(orc, d, g, c, cbg):
    """Per-token optimality: no centroid is closer by more than the fp32
    rounding of the distance itself (float64 brute force, independent)."""
    rng = _rng(d * 1000 + c)
    keys = rng.standard_normal((300, d)).astype(np.float16)
    C = rng.standard_normal((cbg, c, d // g)).astype(np.float32)
    codes = orc.encode(keys, C, g)
    dbar = d // g
    for i in range(g):
        Ci = C[0 if cbg == 1 else i].astype(np.float64)
        sub = keys[:, i * dbar:(i + 1) * dbar].astype(np.float64)
        dist = ((sub[:, None, :] - Ci[None]) ** 2).sum(-1)
        chosen = dist[np.arange(len(keys)), codes[:, i]]
        best = dist.min(1)
        slack = 4 * dbar * 2.0 ** -24 * (best + 1e-30) + 1e-30
        assert np.all(chosen <= best + slack)
        # strictly closer centroids (beyond rounding) with lower index never exist
        assert np.all(codes[:, i] < c)


def test_encode_planted_zero_noise_identity(orc):
    """zero-noise planted keys, c >= clusters -> reconstruct(encode(K)) == K."""
    keys, C, _ = synth.planted_keys(7, 200, 32, 8, clusters=6, cbg_c=16)
    codes = orc.encode(keys, C, 8)
    rec = orc.reconstruct(codes, C, 32)
    assert np.array_equal(rec, keys.astype(np.float32))


def test_encode_reconstruct_idempotent(orc):
    """encode(reconstruct(P)) == P for distinct centroids."""
    rng = _rng(3)
    C = rng.standard_normal((4, 40, 4)).astype(np.float16).astype(np.float32)
    P = rng.integers(0, 40, size=(100, 4)).astype(np.uint16)
    rec = orc.reconstruct(P, C, 16).astype(np.float16)
    assert np.array_equal(orc.encode(rec, C, 4), P)


# ---------------------------------------------------------------- R2 table
def _table_bound(q, C, g):
    d = q.shape[1]
    dbar = d // g
    qf = q.astype(np.float64).reshape(q.shape[0], g, dbar)
    Cf = C.astype(np.float64)
    if Cf.shape[0] == 1:
        Cf = np.repeat(Cf, g, 0)
    exact = np.einsum("hie,ime->him", qf, Cf)
    absum = np.einsum("hie,ime->him", np.abs(qf), np.abs(Cf))
    return exact, dbar * 2.0 ** -24 * absum * 1.0001


@pytest.mark.parametrize("G,d,g,c,cbg", [(4, 128, 32, 256, 32), (2, 64, 16, 100, 1), (1, 16, 1, 37, 1)])
def test_table_fp32_within_rounding_bound(orc, G, d, g, c, cbg):
    """T = q̄·C vs float64 dot products: |T32 - T| <= dbar·u·Σ|q_e C_e| (FMA chain bound).
    g=1 reduces to the dense matrix-vector product q·C₁ᵀ."""
    rng = _rng(G + d + c)
    q = (rng.standard_normal((G, d)) * 2.29).astype(np.float16)
    C = rng.standard_normal((cbg, c, d // g)).astype(np.float32)
    T32, Tfx, e = orc.table(q, C, g)
    exact, bound = _table_bound(q, C, g)
    assert np.all(np.abs(T32 - exact) <= bound + 1e-45)


def test_table_fixed_point_scale_and_rounding(orc):
    """R2 fixed point: the bound A_h (|q̄_i|·max|C| chain) dominates every entry exactly,
    A_h·2^e in [2^14, 2^15), |T_fx - T32·2^e| <= 1/2 (round to nearest); A_h is within
    √dbar·(max over groups of ‖q̄_i‖₁/‖q̄_i‖₂) of the true max (Cauchy-Schwarz)."""
    rng = _rng(11)
    for trial in range(20):
        s = 10.0 ** rng.uniform(-3, 3)
        q = (rng.standard_normal((4, 32)) * s).astype(np.float16)
        C = rng.standard_normal((8, 64, 4)).astype(np.float32)
        T32, Tfx, e = orc.table(q, C, 8)
        Cabs = np.abs(C).max(1)
        assert np.array_equal(orc.codebook_absmax(C), Cabs)
        for h in range(4):
            A = orc.table_bound(q[h], C, 8)
            amax = np.abs(T32[h]).max()
            assert amax <= A
            # independent float64 value of the bound
            A64 = (np.abs(q[h].astype(np.float64)).reshape(8, 4) * Cabs).sum(1).max()
            assert abs(A - A64) <= 4 * 2.0 ** -23 * A64
            if A == 0:
                continue
            scaled = T32[h].astype(np.float64) * 2.0 ** int(e[h])
            assert 2 ** 14 <= A * 2.0 ** int(e[h]) < 2 ** 15
            assert np.all(np.abs(Tfx[h] - scaled) <= 0.5)
            assert np.abs(Tfx[h]).max() <= 32767


def test_table_8bit_variant_scale_and_bound(orc):
    """R2b (8-bit table): A·2^e in [2^6, 2^7), |T_fx| <= 127, round to nearest,
    and the 16-bit table is the same values on a 2^8-finer grid (|T16 - 256·T8| <= 128.5)."""
    rng = _rng(111)
    for trial in range(10):
        q = (rng.standard_normal((4, 128)) * 2.29).astype(np.float16)
        C = rng.standard_normal((32, 256, 4)).astype(np.float32)
        T32, T8, e8 = orc.table(q, C, 32, lut_bits=8)
        _, T16, e16 = orc.table(q, C, 32)
        assert np.array_equal(e16, e8 + 8)
        for h in range(4):
            A = orc.table_bound(q[h], C, 32)
            assert 2 ** 6 <= A * 2.0 ** int(e8[h]) < 2 ** 7
            assert np.abs(T8[h]).max() <= 127
            assert np.all(np.abs(T8[h] - T32[h].astype(np.float64) * 2.0 ** int(e8[h])) <= 0.5)
            assert np.all(np.abs(T16[h].astype(np.int64) - 256 * T8[h].astype(np.int64)) <= 128.5)


def test_table_zero_query(orc):
    """q = 0 -> T = 0 (and the scale falls back to 2^100)."""
    C = _rng(1).standard_normal((4, 16, 2)).astype(np.float32)
    T32, Tfx, e = orc.table(np.zeros((2, 8), np.float16), C, 4)
    assert not T32.any() and not Tfx.any() and list(e) == [100, 100]


def test_scale_exponent_closed_form(orc):
    assert orc.scale_exponent(1.0) == 14
    assert orc.scale_exponent(1.999) == 14
    assert orc.scale_exponent(2.0) == 13
    assert orc.scale_exponent(32767.0) == 0
    assert orc.scale_exponent(0.0) == 100
    assert orc.scale_exponent(2.0 ** -101) == 100
    assert orc.scale_exponent(2.0 ** 120) == -100


# ---------------------------------------------------------------- R3 scores (Eq. 3)
def test_scores_pure_gather_identity(orc):
    """g=1, c=n, P[j]=j -> z[j] = T[0][j]."""
    T = _rng(2).integers(-32767, 32768, size=(1, 500)).astype(np.int16)
    P = np.arange(500, dtype=np.uint16)[None]
    assert np.array_equal(orc.scores(T, P, 500), T[0].astype(np.int32))


def test_scores_brute_force_sum(orc):
    """Eq. 3 z_j = Σ_i T[i][P[j][i]] (numpy int64 gather-sum, independent), strided P."""
    rng = _rng(4)
    g, c, n, stride = 32, 300, 777, 800
    T = rng.integers(-32767, 32768, size=(g, c)).astype(np.int16)
    P = rng.integers(0, c, size=(g, stride)).astype(np.uint16)
    ref = T.astype(np.int64)[np.arange(g)[:, None], P[:, :n]].sum(0)
    assert np.array_equal(orc.scores(T, P, n), ref.astype(np.int32))


@pytest.mark.parametrize("g,dbar,c", [(32, 4, 512), (64, 2, 256), (16, 8, 128)])
def test_scores_equal_dot_with_reconstruction(orc, g, dbar, c):
    """Eq. 2/3 identity (C-P1/C-P4): z̃·2^-e == q·Q(K)_j within the closed-form
    bound g·(2^-e/2 + max FMA-chain error of T)."""
    rng = _rng(g * c)
    d = g * dbar
    q = (rng.standard_normal((4, d)) * 2.29).astype(np.float16)
    C = rng.standard_normal((g, c, dbar)).astype(np.float32)
    P = rng.integers(0, c, size=(g, 1000)).astype(np.uint16)
    T32, Tfx, e = orc.table(q, C, g)
    rec = orc.reconstruct(P.T.copy(), C, d).astype(np.float64)
    _, tb = _table_bound(q, C, g)
    for h in range(4):
        z = orc.scores(Tfx[h], P, 1000).astype(np.float64) * 2.0 ** -int(e[h])
        exact = rec @ q[h].astype(np.float64)
        bound = g * (0.5 * 2.0 ** -int(e[h]) + tb[h].max())
        assert np.max(np.abs(z - exact)) <= bound


def test_resident_scores_exact_dot_bound(orc):
    """Resident tokens: exact fp32 FMA dot onto the 2^-e grid: |z·2^-e - q·k| <= d·u·Σ|q k| + 2^-e/2."""
    rng = _rng(5)
    q = rng.standard_normal(128).astype(np.float16)
    rk = rng.standard_normal((50, 128)).astype(np.float16)
    for e in (0, 7, 14):
        z = orc.resident_scores(q, rk, e).astype(np.float64) * 2.0 ** -e
        exact = rk.astype(np.float64) @ q.astype(np.float64)
        bound = 128 * 2.0 ** -24 * (np.abs(rk.astype(np.float64)) @ np.abs(q.astype(np.float64))) + 0.5 * 2.0 ** -e
        assert np.all(np.abs(z - exact) <= bound)


# ---------------------------------------------------------------- R4 normalise
def test_kappa_closed_form(orc):
    assert orc.kappa(128, 0) == np.float32(math.log2(math.e) / math.sqrt(128))
    assert float(np.float32(orc.kappa(128, 0))).hex() == "0x1.0527dc0000000p-3"
    assert orc.kappa(128, 5) == np.float32(orc.kappa(128, 0)) * np.float32(2.0 ** -5)


def test_exp2_poly_accuracy(orc):
    """exp2_det's polynomial vs the closed form 2^f on [0,1): rel err < 2^-23 (fit: 6.2e-8)."""
    f = np.linspace(0, 1, 20001, endpoint=False).astype(np.float32)
    p = np.array([orc.exp2_poly(float(x)) for x in f], np.float64)
    assert np.max(np.abs(p / np.exp2(f.astype(np.float64)) - 1)) < 2.0 ** -23


def test_mass_closed_form_and_monotone(orc):
    """W(Δ) = floor(2^40·2^{-Δκ}) up to the polynomial error; W(0) = 2^40; non-increasing;
    zero once Δκ > 40."""
    kap = orc.kappa(128, 14)
    assert orc.mass(0, kap) == 2 ** 40
    prev = 2 ** 40
    for delta in list(range(0, 5000, 7)) + list(range(5000, 6_000_000, 9973)):
        W = orc.mass(delta, kap)
        x = -np.float32(np.float32(delta) * np.float32(kap))
        ref = 2.0 ** (40 + float(x))
        if float(x) < -40:
            assert W == 0
        else:
            assert abs(W - ref) <= ref * 2.0 ** -22 + 1.0
        assert W <= prev
        prev = W


def test_threshold_exact_ceiling(orc):
    rng = _rng(9)
    for _ in range(2000):
        tq = int(rng.integers(0, 2 ** 24 + 1))
        S = int(rng.integers(1, 2 ** 62))
        assert orc.threshold(tq, S) == -((-tq * S) // 2 ** 24)

def test_tau_q_single_valued(orc):
    """R5: τ_q = rint(τ·2^24) of the fp32 τ, round-half-even -- one value per τ, worked by
    hand from the fp32 bit patterns (not by re-evaluating the formula)."""
    # fp32(0.9) = 15099494 * 2^-24 exactly (0x3F666666: mantissa 0x666666 | 1<<23 = 15099494,
    # exponent -1 -> 15099494 * 2^-24) -> τ·2^24 is an integer: 15099494
    assert orc.tau_q(0.9) == 15099494
    # fp32(0.3) = 0x3E99999A = 10066330 * 2^-25 -> τ·2^24 = 5033165.0
    assert orc.tau_q(0.3) == 5033165
    # exact half-way points round to even: (2^23 + 1) * 2^-25 -> 2^22 + 0.5 -> 2^22 (even);
    # (2^23 + 3) * 2^-25 -> 2^22 + 1.5 -> 2^22 + 2
    assert orc.tau_q(float(np.float32((2 ** 23 + 1) * 2.0 ** -25))) == 2 ** 22
    assert orc.tau_q(float(np.float32((2 ** 23 + 3) * 2.0 ** -25))) == 2 ** 22 + 2
    assert orc.tau_q(1.0) == 2 ** 24
    assert orc.tau_q(2.0 ** -24) == 1 and orc.tau_q(2.0 ** -26) == 0


def test_select_float_grid_worked_values(orc):
    """R5b grid: e = clamp(21 - floor(log2 max|z|), -100, 100) (100 if max|z| <
    2^-100), z_fx = rint(clamp(z·2^e, ±2^22)); every expected value worked by hand."""
    e, z = orc.float_grid(np.array([1.0], np.float32))            # floor(log2 1) = 0
    assert e == 21 and z.tolist() == [2 ** 21]
    e, z = orc.float_grid(np.array([3.0, -1.5], np.float32))      # floor(log2 3) = 1
    assert e == 20 and z.tolist() == [3 * 2 ** 20, -3 * 2 ** 19]
    e, z = orc.float_grid(np.array([0.75, 0.5], np.float32))      # floor(log2 0.75) = -1
    assert e == 22 and z.tolist() == [3 * 2 ** 20, 2 ** 21]
    # ties to even on the grid: max|z| = 1 -> e = 21; 2.5 and 3.5 grid units -> 2 and 4
    e, z = orc.float_grid(np.array([1.0, 2.5 * 2.0 ** -21, 3.5 * 2.0 ** -21, -2.5 * 2.0 ** -21], np.float32))
    assert e == 21 and z.tolist() == [2 ** 21, 2, 4, -2]
    # 0.1 (fp32 0x3DCCCCCD = 13421773 * 2^-27): e = 21 - (-4) = 25 -> 13421773 / 4 = 3355443.25 -> 3355443
    e, z = orc.float_grid(np.array([0.1], np.float32))
    assert e == 25 and z.tolist() == [3355443]
    # huge scores: floor(log2 3e38) = 127 -> e = -106 clamps to -100; 3e38 * 2^-100 > 2^22 clamps
    e, z = orc.float_grid(np.array([3e38, -3e38, 1.0], np.float32))
    assert e == -100 and z.tolist() == [2 ** 22, -(2 ** 22), 0]
    # tiny scores: max|z| < 2^-100 -> e = 100
    e, z = orc.float_grid(np.array([2.0 ** -110, 0.0], np.float32))  # 2^-110 * 2^100 = 2^-10 -> 0
    assert e == 100 and z.tolist() == [0, 0]
    e, z = orc.float_grid(np.zeros(3, np.float32))
    assert e == 100 and z.tolist() == [0, 0, 0]


def test_select_float_grid_properties(orc):
    """R5b: the largest |z| lands in [2^21, 2^22); every z_fx is within half a grid step of
    z·2^e (no clamping below the 2^22 bound); the grid is monotone (a mis-rounding, a wrong
    exponent or a dropped clamp fails one of these)."""
    rng = _rng(31)
    for trial in range(200):
        scale = float(2.0 ** rng.integers(-60, 60))
        zf = (rng.standard_normal(int(rng.integers(1, 400))) * scale).astype(np.float32)
        e, z = orc.float_grid(zf)
        A = float(np.max(np.abs(zf)))
        if A == 0.0:
            continue
        assert 2 ** 21 <= int(np.max(np.abs(z))) <= 2 ** 22
        exact = zf.astype(np.float64) * 2.0 ** e
        assert np.all(np.abs(z - exact) <= 0.5)
        o = np.argsort(zf, kind="stable")
        assert np.all(np.diff(z[o]) >= 0)
        # selection on the grid is the integer selection at scale e
        r = orc.select_float(zf, 128, 0.9, 1 + trial % 50)
        ri = orc.select(z, e, 128, 0.9, 1 + trial % 50)
        assert r["idx"].tolist() == ri["idx"].tolist() and np.array_equal(r["w"], ri["w"])


# ---------------------------------------------------------------- R5 selection (Eq. 4)
def _brute_select(W, tau_q, k_max):
    """Exhaustive search (C-P5): the smallest cardinality k such that SOME subset
    of size k has mass >= Θ; among those, the max-mass subset, ties -> lexicographically
    lowest sorted index tuple.  Then cap at k_max the same way."""
    n = len(W)
    S = sum(W)
    theta = -((-tau_q * S) // 2 ** 24)
    kstar = n
    if tau_q < 2 ** 24:
        for k in range(1, n + 1):
            if any(sum(W[j] for j in comb) >= theta for comb in itertools.combinations(range(n), k)):
                kstar = k
                break
    ksel = min(kstar, k_max)
    best = None
    for comb in itertools.combinations(range(n), ksel):
        key = (-sum(W[j] for j in comb), comb)
        if best is None or key < best:
            best = key
    return kstar, list(best[1])


def test_select_brute_force_tiny(orc):
    """Eq. 4 on n <= 9 with heavy ties, all τ of Table 3 and several caps vs brute force."""
    rng = _rng(12)
    taus = GOLD["table3_tau_grid"]["taus"]
    kap = orc.kappa(128, 10)
    for trial in range(160):
        n = int(rng.integers(1, 10))
        z = rng.integers(-3000, 3000, size=n) if trial % 2 else rng.integers(-4, 4, size=n) * 500
        z = z.astype(np.int32)
        M = int(z.max())
        W = [orc.mass(M - int(v), kap) for v in z]
        for tau in taus:
            for k_max in (1, 3, n):
                r = orc.select(z, 10, 128, tau, k_max)
                kstar, sel = _brute_select(W, orc.tau_q(tau), k_max)
                assert r["kstar"] == kstar
                assert r["idx"].tolist() == sel


def test_select_spec_examples(orc):
    """uniform 1/10 over n=10, τ=0.5 -> k*=5; τ=1 selects all (Table 3)."""
    z = np.zeros(10, np.int32)
    r = orc.select(z, 0, 128, 0.5, 100)
    assert r["kstar"] == 5 and r["idx"].tolist() == [0, 1, 2, 3, 4]
    r = orc.select(z, 0, 128, 1.0, 100)
    assert r["k_sel"] == 10
    assert abs(r["w"].sum() - 1.0) < 1e-15


def test_select_invariants_random(orc):
    """threshold met, minimality, top-k* property, monotone in τ, τ=1 -> all,
    weights are W/S and sum to 1 over all candidates; shift invariance."""
    rng = _rng(13)
    kap_e = 12
    for trial in range(30):
        n = int(rng.integers(50, 3000))
        z = (rng.standard_normal(n) * 3000).astype(np.int32)
        M = int(z.max())
        kap = orc.kappa(128, kap_e)
        W = np.array([orc.mass(M - int(v), kap) for v in z], dtype=object)
        S = int(sum(W))
        prev = 0
        for tau in (0.3, 0.5, 0.7, 0.9, 0.99, 1.0):
            r = orc.select(z, kap_e, 128, tau, n)
            assert r["S"] == S
            sel = set(r["idx"].tolist())
            tq = orc.tau_q(tau)
            msel = sum(W[j] for j in sel)
            if tq >= 2 ** 24:
                assert len(sel) == n
            else:
                assert msel * 2 ** 24 >= tq * S
                worst = max(sel, key=lambda j: (-z[j], j))
                assert (msel - W[worst]) * 2 ** 24 < tq * S
            unsel = [j for j in range(n) if j not in sel]
            if unsel and sel:
                assert min(z[j] for j in sel) >= max(z[j] for j in unsel)
            assert len(sel) >= prev
            prev = len(sel)
            for j, wj in zip(r["idx"], r["w"]):
                assert wj == float(W[j]) / float(S)
        r1 = orc.select(z, kap_e, 128, 0.9, n)
        r2 = orc.select(z + 777, kap_e, 128, 0.9, n)
        assert r1["idx"].tolist() == r2["idx"].tolist() and np.array_equal(r1["w"], r2["w"])


def test_select_cap(orc):
    rng = _rng(14)
    z = (rng.standard_normal(2000) * 4000).astype(np.int32)
    full = orc.select(z, 12, 128, 0.9, 2000)
    for k_max in (1, 17, full["kstar"] - 1, full["kstar"], full["kstar"] + 5):
        r = orc.select(z, 12, 128, 0.9, k_max)
        assert r["k_sel"] == min(full["kstar"], k_max)
        order = sorted(range(2000), key=lambda j: (-z[j], j))[:r["k_sel"]]
        assert r["idx"].tolist() == sorted(order)


def test_select_weights_match_float64_softmax(orc):
    """ã = softmax(z̃/√d): W_j/S vs float64 softmax of z·2^-e/√d within the closed
    form |w - a| <= a·(e^{2·EXP2_ERR} - 1) + 1/S (relative exp2 error + integer truncation)."""
    rng = _rng(15)
    e = 13
    z = (rng.standard_normal(5000) * 2.29 * math.sqrt(128) * 2 ** e).clip(-2 ** 22, 2 ** 22).astype(np.int32)
    r = orc.select(z, e, 128, 1.0, 5000)
    x = z.astype(np.float64) * 2.0 ** -e / math.sqrt(128)
    sm = np.exp(x - x.max())
    sm /= sm.sum()
    w = np.zeros(5000)
    w[r["idx"]] = r["w"]
    bound = sm * (math.exp(2 * EXP2_ERR) - 1) + 1.0 / r["S"]
    assert np.all(np.abs(w - sm) <= bound)


def test_select_float_spec_examples(orc):
    """uniform scores -> 0.25 each; scores (1000, 0) with d=1 -> (1, 0), no overflow."""
    r = orc.select_float(np.zeros(4, np.float32), 128, 1.0, 4)
    assert np.allclose(r["w"], 0.25, rtol=0, atol=1e-15)
    r = orc.select_float(np.array([1000.0, 0.0], np.float32), 1, 1.0, 2)
    assert r["idx"].tolist() == [0, 1]
    assert r["w"][0] == 1.0 and r["w"][1] == 0.0


# ---------------------------------------------------------------- f4 block-wise prefill (App. B)
def test_blockwise_one_block_is_causal_attention(orc):
    """bs >= n: the anchor block is the whole prompt -> plain causal attention, i.e. Eq. 1
    over the prefix (or_exact_attention, pinned above), per query and head (GQA 2)."""
    rng = _rng(81)
    n, Hq, Hkv, d = 40, 4, 2, 32
    q = rng.standard_normal((n, Hq, d)).astype(np.float16)
    k = rng.standard_normal((n, Hkv, d)).astype(np.float16)
    v = rng.standard_normal((n, Hkv, d)).astype(np.float16)
    out = orc.blockwise_attention(q, k, v, 64)
    for i in (0, 1, 17, 39):
        for h in range(Hq):
            ref = orc.exact_attention(q[i, h], k[: i + 1, h // 2], v[: i + 1, h // 2])
            assert np.allclose(out[i, h], ref, rtol=1e-12, atol=1e-12)


def test_blockwise_anchor_plus_local_keys(orc):
    """Query i of block kb >= 1 sees exactly the anchor block and its own block's prefix:
    equal to Eq. 1 over that gathered key list, and blind to every other key (perturbing
    them leaves the output bit-identical)."""
    rng = _rng(82)
    n, Hq, Hkv, d, bs = 50, 2, 1, 16, 12
    q = rng.standard_normal((n, Hq, d)).astype(np.float16)
    k = rng.standard_normal((n, Hkv, d)).astype(np.float16)
    v = rng.standard_normal((n, Hkv, d)).astype(np.float16)
    out = orc.blockwise_attention(q, k, v, bs)
    for i in (12, 13, 30, 49):
        kb = i // bs
        keys = list(range(bs)) + list(range(kb * bs, i + 1))
        for h in range(Hq):
            ref = orc.exact_attention(q[i, h], k[keys, 0], v[keys, 0])
            assert np.allclose(out[i, h], ref, rtol=1e-12, atol=1e-12)
    k2, v2 = k.copy(), v.copy()
    k2[bs:2 * bs] = rng.standard_normal((bs, Hkv, d))  # block 1: invisible to blocks >= 2
    v2[bs:2 * bs] = rng.standard_normal((bs, Hkv, d))
    out2 = orc.blockwise_attention(q, k2, v2, bs)
    assert np.array_equal(out[2 * bs:], out2[2 * bs:])
    assert not np.array_equal(out[bs:2 * bs], out2[bs:2 * bs])


# ---------------------------------------------------------------- f4 MiniBatchKMeans step
def test_kmeans_first_step_is_cluster_mean_and_matches_sklearn(orc):
    """With v = 0 the step is one Lloyd iteration: every assigned centre becomes the mean of
    its sub-vectors (float64 mean -> fp32, bit for bit) -- and matches scikit-learn's KMeans
    (max_iter=1, the library P:356 uses) within fp32 rounding; unassigned centres stay."""
    from sklearn.cluster import KMeans
    rng = _rng(71)
    d, g, c = 16, 4, 6
    dbar = d // g
    planted = rng.standard_normal((c, dbar)) * 4
    X = (planted[rng.integers(0, c, 3000)] + rng.standard_normal((3000, dbar)) * 0.3)
    keys = X.reshape(750, d).astype(np.float16)  # 750 keys x 4 groups, one shared codebook
    C0 = (planted + rng.standard_normal((c, dbar)) * 0.5).astype(np.float32)[None]
    C1, v1, lab = orc.kmeans_step(keys, C0, np.zeros((1, c), np.int64), np.arange(750), g)
    sub = keys.astype(np.float64).reshape(-1, dbar)
    labs = lab.reshape(-1)
    for m in range(c):
        pts = sub[labs == m]
        assert v1[0, m] == len(pts)
        if len(pts):
            assert np.array_equal(C1[0, m], pts.mean(0).astype(np.float32))
        else:
            assert np.array_equal(C1[0, m], C0[0, m])
    km = KMeans(n_clusters=c, init=C0[0].astype(np.float64), n_init=1, max_iter=1,
                algorithm="lloyd").fit(sub)
    # sklearn reports the centres after its iteration
    assert np.allclose(km.cluster_centers_, C1[0], rtol=1e-5, atol=1e-5)


def test_kmeans_equals_sequential_sculley(orc):
    """The batched update equals Sculley's Alg. 1 (per-sample c <- (1 - 1/v)c + x/v with
    assignments cached at the start of the batch) within fp32 rounding, per-group codebooks,
    non-zero prior counts, repeated sample indices."""
    rng = _rng(72)
    d, g, c = 32, 8, 5
    dbar = d // g
    keys = rng.standard_normal((400, d)).astype(np.float16)
    C0 = rng.standard_normal((g, c, dbar)).astype(np.float32)
    v0 = rng.integers(0, 50, size=(g, c)).astype(np.int64)
    sample = rng.integers(0, 400, size=300)
    C1, v1, lab = orc.kmeans_step(keys, C0, v0, sample, g)
    assert np.array_equal(lab, orc.encode(keys[sample], C0, g))
    C = C0.astype(np.float64).copy()
    v = v0.copy()
    for s_, j in enumerate(sample):
        for i in range(g):
            m = int(lab[s_, i])
            x = keys[j, i * dbar:(i + 1) * dbar].astype(np.float64)
            v[i, m] += 1
            eta = 1.0 / v[i, m]
            C[i, m] = (1 - eta) * C[i, m] + eta * x
    assert np.array_equal(v, v1)
    assert np.allclose(C1, C, rtol=1e-6, atol=1e-6)
    assert v1.sum() - v0.sum() == 300 * g


def test_kmeans_converges_on_planted_clusters(orc):
    """Repeated steps on keys drawn around planted centres recover them (MiniBatchKMeans
    converges; the step is deterministic)."""
    rng = _rng(73)
    d, g, c = 8, 2, 4
    dbar = d // g
    planted = rng.standard_normal((g, c, dbar)) * 5
    lab = rng.integers(0, c, size=(5000, g))
    keys = np.concatenate([planted[i][lab[:, i]] for i in range(g)], 1)
    keys = (keys + rng.standard_normal(keys.shape) * 0.05).astype(np.float16)
    C = (planted + rng.standard_normal(planted.shape) * 1.0).astype(np.float32)
    v = np.zeros((g, c), np.int64)
    for it in range(20):
        C, v, _ = orc.kmeans_step(keys, C, v, rng.integers(0, 5000, size=500), g)
    for i in range(g):
        err = np.linalg.norm(np.sort(C[i], 0) - np.sort(planted[i], 0))
        assert err < 0.1
    a = orc.kmeans_step(keys, C, v, np.arange(100), g)
    b = orc.kmeans_step(keys, C, v, np.arange(100), g)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


# ---------------------------------------------------------------- R8 shared selection (f3(iii))
def _shared_A(orc, z, e, d=128):
    """Â_{h,j} = floor(W_{h,j}·ρ_h / 2^64), ρ_h = floor((2^104-1)/S_h), A_j = Σ_h Â_{h,j} in
    Python integers (R8), on the pinned R4 masses."""
    G, n = z.shape
    A = [0] * n
    for h in range(G):
        kap = orc.kappa(d, int(e[h]))
        M = int(z[h].max())
        W = [orc.mass(M - int(v), kap) for v in z[h]]
        rho = ((1 << 104) - 1) // sum(W)
        for j in range(n):
            A[j] += (W[j] * rho) >> 64
    return A


def test_select_shared_brute_force_tiny(orc):
    """R8 on n <= 8, G in {2, 4}, heavy ties: the kept set is the exhaustive minimal prefix of
    the head-averaged mass A (brute force over all subsets, C-P5's rule on A)."""
    rng = _rng(61)
    for trial in range(80):
        G = 2 if trial % 2 else 4
        n = int(rng.integers(1, 9))
        z = (rng.integers(-3, 3, size=(G, n)) * 700 if trial % 3 == 0
             else rng.integers(-3000, 3000, size=(G, n))).astype(np.int32)
        e = rng.integers(9, 12, size=G).astype(np.int32)
        A = _shared_A(orc, z, e)
        for tau in (0.3, 0.6, 0.9, 1.0):
            for k_max in (1, 3, n):
                r = orc.select_shared(z, e, 128, tau, k_max)
                assert r["A"].tolist() == A
                kstar, sel = _brute_select(A, orc.tau_q(tau), k_max)
                assert r["kstar"] == kstar
                assert r["idx"].tolist() == sel


def test_select_shared_mass_is_mean_softmax(orc):
    """A_j / (G·2^40) = (1/G) Σ_h softmax_h(z̃/√d)_j within the closed form per head
    a·(e^{2·EXP2_ERR} - 1) + 1/S_h + 2^-40 + 2^-63 (exp2 error, W truncation, ρ and Â
    floors); S_A within [G·(2^40 - n - 1), G·(2^40 - 1)]."""
    rng = _rng(62)
    G, n = 4, 3000
    e = np.array([12, 13, 12, 14], np.int32)
    z = np.stack([(rng.standard_normal(n) * 2.29 * math.sqrt(128) * 2.0 ** int(e[h]))
                  .clip(-2 ** 22, 2 ** 22) for h in range(G)]).astype(np.int32)
    r = orc.select_shared(z, e, 128, 1.0, n)
    assert r["k_sel"] == n
    SA = r["S_A"]
    assert G * (2 ** 40 - n - 1) <= SA <= G * (2 ** 40 - 1)
    assert SA == int(sum(int(a) for a in r["A"]))
    mean = np.zeros(n)
    bound = np.zeros(n)
    for h in range(G):
        x = z[h].astype(np.float64) * 2.0 ** -int(e[h]) / math.sqrt(128)
        sm = np.exp(x - x.max())
        sm /= sm.sum()
        S_h = sum(orc.mass(int(z[h].max()) - int(v), orc.kappa(128, int(e[h]))) for v in z[h])
        mean += sm / G
        bound += (sm * (math.exp(2 * EXP2_ERR) - 1) + 1.0 / S_h + 2.0 ** -40 + 2.0 ** -63) / G
    got = r["A"].astype(np.float64) / (G * 2.0 ** 40)
    assert np.all(np.abs(got - mean) <= bound)


def test_select_shared_invariants(orc):
    """R8: threshold met and minimal on A, top-k* by (A desc, index asc), monotone in τ,
    τ = 1 -> all, the cap keeps the A-order prefix, n = 1 keeps {0} with weight 1."""
    rng = _rng(63)
    G, n = 4, 1500
    e = np.full(G, 12, np.int32)
    z = (rng.standard_normal((G, n)) * 3000).astype(np.int32)
    prev = 0
    order = None
    for tau in (0.2, 0.5, 0.9, 0.99, 1.0):
        r = orc.select_shared(z, e, 128, tau, n)
        A = [int(a) for a in r["A"]]
        order = sorted(range(n), key=lambda j: (-A[j], j))
        sel = r["idx"].tolist()
        assert sel == sorted(order[:r["k_sel"]])
        tq = orc.tau_q(tau)
        m = sum(A[j] for j in sel)
        if tq >= 2 ** 24:
            assert len(sel) == n
        else:
            assert m * 2 ** 24 >= tq * r["S_A"]
            assert (m - A[order[r["k_sel"] - 1]]) * 2 ** 24 < tq * r["S_A"]
        assert len(sel) >= prev
        prev = len(sel)
    full = orc.select_shared(z, e, 128, 0.9, n)
    for k_max in (1, 10, full["kstar"] - 1, full["kstar"]):
        r = orc.select_shared(z, e, 128, 0.9, k_max)
        assert r["k_sel"] == min(k_max, full["kstar"])
        assert r["idx"].tolist() == sorted(order[:r["k_sel"]]) or k_max >= full["kstar"]
    r = orc.select_shared(np.array([[5], [-7]], np.int32), np.array([3, 4], np.int32), 128, 0.9, 4)
    assert r["idx"].tolist() == [0] and np.all(r["w"] == 1.0)


def test_decode_shared_tau1_equals_per_head(orc):
    """R8 at τ = 1 keeps every token, so each head's Eq. 5 output equals the per-head
    decode's bit for bit (same weights W/S, same ascending summation)."""
    rng = _rng(64)
    G, d, g, c, n = 4, 128, 32, 64, 700
    q = (rng.standard_normal((G, d)) * 2.0).astype(np.float16)
    C_ = rng.standard_normal((g, c, d // g)).astype(np.float32)
    P = rng.integers(0, c, size=(g, n)).astype(np.uint16)
    V = rng.standard_normal((n, d)).astype(np.float16)
    a = orc.decode_unit(q, C_, P, n, V, 1.0, n)
    b = orc.decode_unit(q, C_, P, n, V, 1.0, n, shared=True)
    assert np.array_equal(a["out"], b["out"])
    b9 = orc.decode_unit(q, C_, P, n, V, 0.9, n, shared=True)
    assert all(np.array_equal(b9["idx"][0], b9["idx"][h]) for h in range(G))
    assert b9["k_sel"][0] < n


# ---------------------------------------------------------------- R6 gather (Eq. 5)
def test_gather_singleton_is_row(orc):
    """singleton selection (index i, weight 1) -> V_i exactly."""
    V = _rng(16).standard_normal((30, 128)).astype(np.float16)
    out = orc.gather(np.array([7], np.int32), np.array([1.0]), V)
    assert np.array_equal(out, V[7].astype(np.float64))


def test_decode_n1_is_v0(orc):
    """n=1 cache -> output = V_0 for every head regardless of q."""
    rng = _rng(17)
    q = (rng.standard_normal((4, 128)) * 5).astype(np.float16)
    C = rng.standard_normal((32, 64, 4)).astype(np.float32)
    P = rng.integers(0, 64, size=(32, 8)).astype(np.uint16)
    V = rng.standard_normal((1, 128)).astype(np.float16)
    r = orc.decode_unit(q, C, P, 1, V, 0.9, 5)
    for h in range(4):
        assert np.array_equal(r["out"][h], V[0].astype(np.float64))


# exp2_det error budget (natural-log units): x = -(Δ·κ) is rounded once (|x| <= 41 while W > 0)
# and κ is an fp32 rounding of log2(e)/√d (another |x|·2^-24), the polynomial adds < 2^-23.
EXP2_ERR = 41 * 2.0 ** -23 * math.log(2) + 2.0 ** -23


def _output_bound(z_err_nat, vmax, n):
    """Closed-form: logits off by <= eps (natural units) -> each softmax weight off by a factor
    in [e^-2eps, e^2eps]; truncating W to an integer adds <= n/S <= n·2^-40 absolute mass."""
    eps = z_err_nat + EXP2_ERR
    return (math.exp(2 * eps) - 1) * vmax + n * 2.0 ** -39 * vmax


def test_exact_equivalence_planted_integer(orc):
    """C-P2 / SPEC S:439: zero quantization error (planted integer keys/centroids), τ=1 ->
    decode output == exact attention (Eq. 1, float64) within the closed-form bound of the
    fixed-point/exp2 roundings (here T is exact, so only exp2+mass truncation remain)."""
    rng = _rng(18)
    d, g, c, n = 64, 16, 32, 700
    dbar = d // g
    C = rng.integers(-3, 4, size=(g, c, dbar)).astype(np.float32)
    codes = rng.integers(0, c, size=(n, g)).astype(np.uint16)
    K = orc.reconstruct(codes, C, d).astype(np.float16)
    q = rng.integers(-2, 3, size=(4, d)).astype(np.float16)
    V = rng.standard_normal((n, d)).astype(np.float16)
    P = np.ascontiguousarray(codes.T)
    r = orc.decode_unit(q, C, P, n, V, 1.0, n)
    for h in range(4):
        ref = orc.exact_attention(q[h], K, V)
        vmax = float(np.abs(V.astype(np.float64)).max())
        assert np.max(np.abs(r["out"][h] - ref)) <= _output_bound(0.0, vmax, n)


def test_exact_equivalence_planted_gaussian(orc):
    """C-P2 with real-valued planted centres: error within the closed-form bound."""
    keys, C, _ = synth.planted_keys(21, 1500, 128, 32, clusters=20, cbg_c=64)
    rng = _rng(19)
    q = (rng.standard_normal((4, 128)) * 2.29).astype(np.float16)
    codes = orc.encode(keys, C, 32)
    V = rng.standard_normal((1500, 128)).astype(np.float16)
    r = orc.decode_unit(q, C, np.ascontiguousarray(codes.T), 1500, V, 1.0, 1500)
    vmax = float(np.abs(V.astype(np.float64)).max())
    _, tb = _table_bound(q, C, 32)
    for h in range(4):
        ref = orc.exact_attention(q[h], keys, V)
        zerr = (32 * (0.5 * 2.0 ** -int(r["e"][h]) + tb[h].max())) / math.sqrt(128)
        assert np.max(np.abs(r["out"][h] - ref)) <= _output_bound(zerr, vmax, 1500)


def test_vo_only_equivalence_resident(orc):
    """C-P3 / SPEC S:440: value-offload-only (exact keys, all tokens resident), τ=1 ->
    exact attention within the closed-form bound of the fp32 dot + fixed-point grid."""
    rng = _rng(20)
    d = 128
    K = rng.standard_normal((600, d)).astype(np.float16)
    V = rng.standard_normal((600, d)).astype(np.float16)
    q = (rng.standard_normal((4, d)) * 2.29).astype(np.float16)
    C = rng.standard_normal((32, 16, 4)).astype(np.float32)
    P = np.zeros((32, 8), np.uint16)
    r = orc.decode_unit(q, C, P, 0, np.zeros((1, d), np.float16), 1.0, 600, rk=K, rv=V)
    vmax = float(np.abs(V.astype(np.float64)).max())
    for h in range(4):
        ref = orc.exact_attention(q[h], K, V)
        dot_err = d * 2.0 ** -24 * float((np.abs(K.astype(np.float64)) @ np.abs(q[h].astype(np.float64))).max())
        zerr = (dot_err + 0.5 * 2.0 ** -int(r["e"][h])) / math.sqrt(d)
        assert np.max(np.abs(r["out"][h] - ref)) <= _output_bound(zerr, vmax, 600)


def test_decode_deterministic_and_weights_sum(orc):
    """C-P9: run twice -> bit-identical; τ=1 weights sum to 1 (W/S)."""
    rng = _rng(22)
    q = (rng.standard_normal((4, 128)) * 2.29).astype(np.float16)
    C = rng.standard_normal((32, 128, 4)).astype(np.float32)
    P = rng.integers(0, 128, size=(32, 900)).astype(np.uint16)
    V = rng.standard_normal((900, 128)).astype(np.float16)
    a = orc.decode_unit(q, C, P, 900, V, 0.9, 300)
    b = orc.decode_unit(q, C, P, 900, V, 0.9, 300)
    assert np.array_equal(a["out"], b["out"]) and all(np.array_equal(x, y) for x, y in zip(a["idx"], b["idx"]))
    c1 = orc.decode_unit(q, C, P, 900, V, 1.0, 900)
    for h in range(4):
        assert abs(c1["w"][h].sum() - 1.0) < 1e-12


# ---------------------------------------------------------------- paper closed forms
def test_table1a_memory_budget():
    from accounting import memory_budget
    g = GOLD["table1a_memory_budget"]
    for row in g["rows"]:
        if not row["value_offloaded"] and row["g"] is None:
            r = memory_budget(g["d"], None, False)
        else:
            r = memory_budget(g["d"], row["g"], row["value_offloaded"])
        assert (r.K, r.V, r.total) == (row["K"], row["V"], row["total"])


def test_comm_overhead_102_4_MB():
    from accounting import comm_overhead
    c = GOLD["comm_overhead"]
    b = comm_overhead(c["n"], c["L"], c["H"], c["retain_fraction"], c["bytes_per_score"])
    assert b == c["bytes"] and b / 1e6 == c["MB"]


def test_cost_per_query_table1b():
    from accounting import cost_per_query
    for case in GOLD["table1b_cost_per_query"]["cases"]:
        r = cost_per_query(case["n"], case["d"], case["c"], case["g"])
        assert r == dict(exact_mults=case["exact_mults"], approx_mults=case["approx_mults"],
                         approx_adds=case["approx_adds"])


# ---------------------------------------------------------------- synth generator
def test_synth_splitmix_reference_values():
    """splitmix64 first outputs for seed 0 (Vigna's published 0xe220a8397b1dcdaf,
    0x6e789e6aa1b965f4) and a pure-Python big-int re-derivation for the rest."""
    out = synth.u64(0, 0, 64)
    assert [hex(int(x)) for x in out[:2]] == ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4"]
    M = (1 << 64) - 1

    def fin(z):
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    assert [int(x) for x in out] == [fin((k * 0x9E3779B97F4A7C15) & M) for k in range(1, 65)]


def test_synth_codes_in_range_and_uniform():
    c = 8192
    x = synth.gen_codes(1, 0, 0, 0, 2, c, 0, 200000)
    assert x.max() < c
    h = np.bincount(x[0].astype(np.int64) // 1024, minlength=8)
    assert np.all(np.abs(h / h.sum() - 1 / 8) < 0.01)


def test_synth_value_rows_match_gen_values():
    """synth.gen_value_rows (kept rows only, for huge stores) draws the same counters as
    gen_values row for row."""
    import synth
    full = synth.gen_values(77, 1, 2, 3, 128, 0, 3000)
    rows = np.array([0, 1, 2999, 1234, 17, 17], np.int64)
    assert np.array_equal(synth.gen_value_rows(77, 1, 2, 3, 128, rows).view(np.uint16),
                          full[rows].view(np.uint16))
    part = synth.gen_values(77, 1, 2, 3, 128, 1000, 500)
    assert np.array_equal(synth.gen_value_rows(77, 1, 2, 3, 128, np.arange(1000, 1500)).view(np.uint16),
                          part.view(np.uint16))


def test_oracle_unit_rows_equals_decode_unit():
    """The composed full-size oracle (harness.oracle_unit_rows: kept value rows generated on
    demand) is the oracle's decode_unit, stage for stage."""
    from harness import Case, oracle_unit, oracle_unit_rows
    case = Case(B=1, Hkv=2, n=20011, k_max=1500, tau=0.9, seed=5)
    for kv in range(2):
        a, b = oracle_unit(case, 0, 0, kv), oracle_unit_rows(case, 0, 0, kv, chunk=700)
        assert np.array_equal(a["z"], b["z"]) and np.array_equal(a["S"], b["S"])
        for h in range(case.G):
            assert np.array_equal(a["idx"][h], b["idx"][h]) and np.array_equal(a["w"][h], b["w"][h])
            assert int(a["k_sel"][h]) == int(b["k_sel"][h]) and int(a["kstar"][h]) == int(b["kstar"][h])
        assert np.allclose(a["out"], b["out"], rtol=1e-12, atol=1e-13)
