"""The FAST raster's certified q' error bound, checked by emulation on the CPU.

The raster decides alpha >= theta (rasterize.py:146-151, 209: q <= q_th) from
q' = log2(e) q / 2 evaluated in fp32 (raster_fast.cu quad_q) against a bracket
widened by |q'32 - q'| <= e0q + e1q q' (preprocess.cu write_raster_record).
Every discrete output's bit-exactness rests on that bound, so this test
replays quad_q's exact fp32 operation sequence (each op correctly rounded:
sums and products of float32 are exact in float64 / long double before the
single rounding to float32) on adversarial splats -- elongated and rotated
conics, means anywhere on a 4K screen with non-representable fp64 parts,
pixels inside and around the alpha region -- and compares it with q' in long
double.  The derived bound (without the 1.25 safety factor and the 1.001
widening the product applies) must hold on every sample.
"""
import numpy as np

K = 0.72134752044448170368  # log2(e) / 2
U = 2.0 ** -24
f32, f64, ld = np.float32, np.float64, np.longdouble


def _r32(x):
    return np.asarray(x).astype(f32)


def fadd(a, b):
    return _r32(a.astype(f64) + b.astype(f64))  # exact in fp64 for float32 operands within 2^29 of each other


def fmul(a, b):
    return _r32(a.astype(f64) * b.astype(f64))  # 48-bit product: exact in fp64


def fma(a, b, c):
    return _r32(a.astype(ld) * b.astype(ld) + c.astype(ld))  # one rounding (64-bit mantissa holds the sum)


def _splats(rng, n):
    """Conics of projected 3DGS covariances (+0.3 px^2 dilation), rotated, anisotropy up to ~1e7."""
    s1 = np.exp(rng.uniform(np.log(0.02), np.log(800.0), n))
    s2 = np.exp(rng.uniform(np.log(0.02), np.log(800.0), n))
    th = rng.uniform(0, np.pi, n)
    # a quarter of the splats axis-aligned (the cancellation term vanishes there)
    th[: n // 4] = rng.choice([0.0, np.pi / 2], n // 4)
    c, s = np.cos(th), np.sin(th)
    cxx = c * c * s1 ** 2 + s * s * s2 ** 2 + 0.3
    cyy = s * s * s1 ** 2 + c * c * s2 ** 2 + 0.3
    cxy = c * s * (s1 ** 2 - s2 ** 2)
    det = cxx * cyy - cxy * cxy
    ca, cb, cc = cyy / det, -cxy / det, cxx / det
    m0 = rng.uniform(-200.0, 4040.0, n)
    m1 = rng.uniform(-200.0, 2360.0, n)
    o = rng.uniform(1.0 / 255.0, 1.0, n)
    qth = 2.0 * np.log(o * 255.0)
    return ca, cb, cc, m0, m1, qth


def _record(ca, cb, cc, m0, m1):
    """The raster record fields quad_q reads (write_raster_record)."""
    det = ca * cc - cb * cb
    l11 = np.sqrt(K * ca)
    l21 = K * cb / l11
    l22 = np.sqrt(np.maximum(K * det / ca, 0.0))
    l11f, l21f, l22f = _r32(l11), _r32(l21), _r32(l22)
    mxh, myh = _r32(m0), _r32(m1)
    mxl, myl = m0 - mxh.astype(f64), m1 - myh.astype(f64)
    cu = _r32(l11f.astype(f64) * mxl + l21f.astype(f64) * myl)
    cw = _r32(l22f.astype(f64) * myl)
    return dict(l11=l11f, l21=l21f, l22=l22f, mxh=mxh, myh=myh, cu=cu, cw=cw, det=det)


def _quad_q(r, lx, ly):
    """raster_fast.cu quad_q for one pixel, op by op."""
    dx = fadd(lx, -r["mxh"])
    dy = fadd(ly, -r["myh"])
    t = fma(r["l21"], dy, -r["cu"])
    w = fma(r["l22"], dy, -r["cw"])
    ww = fmul(w, w)
    u = fma(r["l11"], dx, t)
    return fma(u, u, ww)


def _derived_bound(ca, cb, cc, qth, q):
    """e0q + e1q q' of write_raster_record without its 1.25 / 1.001 safety factors."""
    det = ca * cc - cb * cb
    tr = ca + cc
    qt = K * qth
    P = np.sqrt(K * tr)
    sq = np.maximum(np.sqrt(qt), 1e-3)
    bsd = np.abs(cb) / np.sqrt(np.maximum(det, 1e-300))
    e0q = 3.0 * U * P * sq
    e1q = U * (8.0 + 5.0 * bsd) + 3.0 * U * P / sq
    return e0q + e1q * q


def test_fp32_q_bound_holds_on_adversarial_splats():
    rng = np.random.default_rng(2503)
    n = 200_000
    ca, cb, cc, m0, m1, qth = _splats(rng, n)
    rec = _record(ca, cb, cc, m0, m1)
    # pixels: points of the ellipse q' <= 1.3 q_th' mapped through the inverse Cholesky factor, snapped to
    # the pixel centre, on screen
    rad = np.sqrt(K * qth * 1.3) * np.sqrt(rng.uniform(0, 1, n))
    ang = rng.uniform(0, 2 * np.pi, n)
    uu, ww = rad * np.cos(ang), rad * np.sin(ang)
    l11 = np.sqrt(K * ca)
    l21 = K * cb / l11
    l22 = np.sqrt(np.maximum(K * (ca * cc - cb * cb) / ca, 0.0))
    dy = ww / l22
    dx = (uu - l21 * dy) / l11
    px = np.clip(np.floor(m0 + dx), 0, 3839) + 0.5
    py = np.clip(np.floor(m1 + dy), 0, 2159) + 0.5
    q32 = _quad_q(rec, _r32(px), _r32(py)).astype(ld)
    ddx, ddy = px.astype(ld) - m0.astype(ld), py.astype(ld) - m1.astype(ld)
    q = ld(K) * (ca.astype(ld) * ddx * ddx + 2 * cb.astype(ld) * ddx * ddy + cc.astype(ld) * ddy * ddy)
    err = np.abs(q32 - q).astype(f64)
    bound = _derived_bound(ca, cb, cc, qth, q.astype(f64))
    ratio = err / bound
    worst = int(np.argmax(ratio))
    assert ratio.max() <= 1.0, (ratio.max(), ca[worst], cb[worst], cc[worst], m0[worst], m1[worst], px[worst],
                                py[worst], float(q[worst]), err[worst], bound[worst])
    # the bound is not vacuous: near-threshold samples use a sizeable part of it
    near = (q.astype(f64) > 0.5 * K * qth) & (q.astype(f64) < 1.3 * K * qth)
    assert ratio[near].max() > 0.05


def test_cancellation_term_vanishes_for_axis_aligned():
    """b = 0: the bound's e1q is the 8u of the coefficient and product roundings (plus the P term)."""
    ca, cb, cc, qth = np.array([0.5]), np.array([0.0]), np.array([0.02]), np.array([2 * np.log(255.0)])
    b = _derived_bound(ca, cb, cc, qth, np.array([1.0]))
    P = np.sqrt(K * 0.52)
    sq = np.sqrt(K * qth[0])
    assert np.isclose(b[0], 3 * U * P * sq + U * 8.0 + 3 * U * P / sq)


def _round_dir(x, up):
    """x (long double) rounded to float32 toward +inf (up) or -inf."""
    r = _r32(x)
    rl = r.astype(ld)
    if up:
        return np.where(rl < x, np.nextafter(r, f32(np.inf)), r)
    return np.where(rl > x, np.nextafter(r, f32(-np.inf)), r)


def test_transmittance_bound_holds_under_adversarial_alpha_errors():
    """raster_fast.cu blend step: T32 and the lower bound L = T32 - D of the exact transmittance.

    Every step's q'32 sits at the edge of the certified q' error (both signs) and ex2.approx at the edge of
    its 2^-21.5 relative error; the reference alpha is min(o 2^-q', 0.99) in fp64 and T the fp64 product
    (rasterize.py:146-177).  40 % of the steps do not blend (m = 0: T unchanged, D grows by 1e-7 T).  After
    every step L <= T <= 2 T32 - L (the kernel's live / done tests) must hold.
    """
    rng = np.random.default_rng(5168)
    n_pix, n_steps = 4096, 1000
    W = 1.001
    T32 = np.ones(n_pix, f32)
    L = np.ones(n_pix, f32)
    T = np.ones(n_pix, f64)
    mode = np.arange(n_pix) % 3  # 0: errors push alpha up, 1: down, 2: random signs per step
    worst = 0.0
    for step in range(n_steps):
        ca, cb, cc, _, _, qth = _splats(rng, n_pix)
        o = rng.uniform(1.0 / 255.0, 1.0, n_pix)
        o[rng.uniform(0, 1, n_pix) < 0.05] = rng.uniform(0.99, 1.0)  # the alpha clamp
        qth = 2.0 * np.log(o * 255.0)
        qt = K * qth
        det, tr = ca * cc - cb * cb, ca + cc
        P = W * np.sqrt(K * tr)
        sq = np.maximum(np.sqrt(qt), 1e-3)
        bsd = np.abs(cb) / np.sqrt(det)
        e0q = W * 1.25 * 3.0 * U * P * sq
        e1q = W * 1.25 * (U * (8.0 + 5.0 * bsd) + 3.0 * U * P / sq)
        e0r = _r32(W * (4.7e-7 + np.log(2.0) * e0q) * (1.0 + 1.0 / 1024.0))
        e1r = _r32(W * np.log(2.0) * e1q * (1.0 + 1.0 / 1024.0))
        qp = rng.uniform(0.0, 1.0, n_pix) ** 2 * qt  # exact q' of a passing pixel (alpha >= theta)
        sgn = np.where(mode == 0, -1.0, np.where(mode == 1, 1.0, rng.choice([-1.0, 1.0], n_pix)))
        dq = (e0q + e1q * qp) / (1.25 * W) * 0.999  # the derived bound's edge (test_fp32_q_bound_...)
        q32 = np.maximum(_r32(qp + sgn * dq), f32(0))
        ex = _r32(np.exp2(-q32.astype(f64)) * (1.0 - sgn * 2.0 ** -21.5 * 0.999))
        al = fmul(_r32(o), ex)
        al = np.where(_r32(o) > f32(0.99), np.minimum(al, f32(0.99)), al)
        E = fma(e1r, q32, e0r)
        m = (rng.uniform(0, 1, n_pix) < 0.6).astype(f32)  # 0: a live step that does not blend
        am = fmul(al, m)
        wgt = fmul(T32, am)
        omm = fadd(np.ones_like(al), -am)
        c7 = _round_dir(T32.astype(ld) * ld(f32(1e-7)), up=True)
        t1 = fadd(T32, -wgt)
        te = _round_dir(wgt.astype(ld) * E.astype(ld) + c7.astype(ld), up=True)
        l1 = _round_dir(L.astype(ld) * omm.astype(ld) - te.astype(ld), up=False)
        T = np.where(m > 0, T * (1.0 - np.minimum(o * np.exp2(-qp), 0.99)), T)
        T32, L = t1, l1
        upper = _round_dir(2.0 * T32.astype(ld) - L.astype(ld), up=True).astype(f64)
        assert np.all(L.astype(f64) <= T), step
        assert np.all(T <= upper), step
        live = T > 1e-30
        if live.any():
            worst = max(worst, float(np.max(np.abs(T32.astype(f64) - T)[live] / (T32 - L).astype(f64)[live])))
    print("worst |T32 - T| / D:", worst)
    assert worst > 0.01  # the adversarial errors reach a visible part of D
