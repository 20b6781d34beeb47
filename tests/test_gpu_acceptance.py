"""Reference acceptance criteria 3, 5 and 9 and the OFDM checks, on the device.

Restates T/test_acceptance.py:81-99 (criterion 3, Fresnel pins and
passivity), :122-175 (criterion 5, two-ray material gradients and the
region-power yaw gradient at 5 operating points), :255-274 (criterion 9,
Doppler) and T/test_channel.py:110-120 (two-path OFDM ripple) through this
package's CUDA path.  Golden values: tests/golden/criteria.npz, written by
running the reference (make_golden.py criteria_case).
"""

import cmath
import math

import numpy as np
import pytest
import torch

import oracle as O
from conftest import golden_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2303_11103_b200 as P
    assert torch.cuda.is_available()
    return P


def test_criterion_03_fresnel_pins_and_passivity(P):
    rng = np.random.RandomState(2024)
    etas = [rng.uniform(1.0, 50.0) for _ in range(100)]
    te, tm = P.fresnel_batch(np.array(etas, dtype=np.complex128), np.ones(100))
    want = np.array([(1 - math.sqrt(e)) / (1 + math.sqrt(e)) for e in etas])
    assert np.abs(te - want).max() < 1e-12 and np.abs(tm - want).max() < 1e-12
    eta, cos = [], []
    for _ in range(10_000):   # the reference's draw order: eta real, eta imag, cos
        re = rng.uniform(1, 80)
        eta.append(complex(re, -rng.uniform(0, 500)))
        cos.append(rng.uniform(0, 1))
    te, tm = P.fresnel_batch(np.array(eta), np.array(cos))
    assert max(np.abs(te).max(), np.abs(tm).max()) <= 1.0 + 1e-12
    # the scalar form used by the reference's callers
    r_te, r_tm = P.fresnel(complex(9.0, -1.0), 0.3)
    bte, btm = P.fresnel_batch([complex(9.0, -1.0)], [0.3])
    assert isinstance(r_te, P.DiffComplex)
    assert r_te.to_complex() == bte[0] and r_tm.to_complex() == btm[0]


def test_criterion_05_gradients_vs_tape_and_fd(P, golden):
    g = golden("criteria")
    sc = golden_scene(g, "two_ray")
    bvh = P.build(sc)
    ps = P.compute_paths(sc, bvh, 1)
    refl = [p for p in ps.paths if p.kind == "specular"][0]
    tx, rx = sc.device("tx"), sc.device("rx")
    mats = P.path_materials(sc, bvh, refl)
    geom = P.geometry_from_path(refl)
    dev = torch.device("cuda", torch.cuda.current_device())

    def refl_power(eps, sig):
        ctx = P.EvalContext(sc, material_values={"ground": (eps, sig)})
        z = P.transfer(ctx, geom, mats, tx, rx, "iso", "iso", math.pi / 2, math.pi / 2)
        return z.abs2() if isinstance(z, P.DiffComplex) else z.real ** 2 + z.imag ** 2

    worst = 0.0
    for (eps0, sig0), (v_ref, ge_ref, gs_ref) in zip(g["mat_points"], g["mat_out"]):
        e = torch.tensor(eps0, dtype=torch.float64, device=dev, requires_grad=True)
        s = torch.tensor(sig0, dtype=torch.float64, device=dev, requires_grad=True)
        v = refl_power(e, s)
        v.backward()
        assert abs(float(v) - v_ref) <= 1e-9 * v_ref
        assert abs(float(e.grad) - ge_ref) <= 1e-6 * abs(ge_ref)
        assert abs(float(s.grad) - gs_ref) <= 1e-6 * abs(gs_ref)
        he, hs = 1e-4 * eps0, 1e-4 * sig0
        fd_e = (refl_power(eps0 + he, sig0) - refl_power(eps0 - he, sig0)) / (2 * he)
        fd_s = (refl_power(eps0, sig0 + hs) - refl_power(eps0, sig0 - hs)) / (2 * hs)
        worst = max(worst, abs(float(e.grad) - fd_e) / abs(fd_e), abs(float(s.grad) - fd_s) / abs(fd_s))
    # region power vs tx yaw, directive tx (tr38901), frozen topology
    sd = golden_scene(g, "dir_scene")
    bd = P.build(sd)
    cell = g["cell"]
    _, frozen = P.point_path_gain(sd, bd, sd.device("tx"), cell, 1)

    def region_power(yaw):
        ctx = P.EvalContext(sd, orientations={"tx": (yaw, 0.0, 0.0)})
        val, _ = P.point_path_gain(sd, bd, sd.device("tx"), cell, 1, ctx=ctx, frozen_paths=frozen)
        return val

    for yaw0, (v_ref, gy_ref) in zip(g["yaw_points"], g["yaw_out"]):
        y = torch.tensor(float(yaw0), dtype=torch.float64, device=dev, requires_grad=True)
        v = region_power(y)
        v.backward()
        assert abs(float(v) - v_ref) <= 1e-9 * v_ref
        assert abs(float(y.grad) - gy_ref) <= 1e-6 * abs(gy_ref)
        h = 1e-6
        fd = (region_power(float(yaw0) + h) - region_power(float(yaw0) - h)) / (2 * h)
        worst = max(worst, abs(float(y.grad) - fd) / abs(fd))
    assert worst < 1e-3, worst


def test_criterion_09_doppler(P, golden):
    g = golden("criteria")
    fs = golden_scene(g, "free_space")
    bvh = P.build(fs)
    ps = P.compute_paths(fs, bvh, 1)
    static = P.apply_doppler(P.compute_gains(fs, bvh, ps), 1e6, 14)
    a_static = static.entries[0].a[0, 0, :]
    assert np.all(a_static == a_static[0])
    moving = P.apply_doppler(P.compute_gains(fs, bvh, ps), 1e6, 14, tx_velocities=[3, 0, 0])
    a = moving.entries[0].a[0, 0, :]
    assert len(a) == 14
    phase = np.unwrap(np.angle(a))
    slope_hz = float(np.polyfit(moving.sample_times, phase, 1)[0] / (2 * math.pi))
    assert abs(slope_hz - 35.02) < 0.1
    assert np.abs(a - g["doppler_a"]).max() <= 1e-9 * np.abs(g["doppler_a"]).max()
    assert np.array_equal(np.asarray(moving.sample_times), g["doppler_t"])


def _cir(P, a, tau):
    a = np.asarray(a, dtype=np.complex128).reshape(1, 1, 1, 1, -1, 1)
    tau = np.asarray(tau, dtype=np.float64).reshape(1, 1, -1)
    return P.Cir(a=a, tau=tau, rx_names=["rx"], tx_names=["tx"], sample_times=np.zeros(1))


def test_ofdm_two_path_ripple_closed_form(P):
    # T/test_channel.py:110-120: delays put the interference extremes on the grid
    n, df = 128, 30e3
    dtau = 2.0 / (n * df)
    f0 = P.subcarrier_frequencies(n, df)[0]
    a1 = 1.0
    a2 = 0.4 * cmath.exp(-2j * math.pi * f0 * dtau)
    fr = P.frequency_response(_cir(P, [a1, a2], [0.0, dtau]), n, df)
    mag = np.abs(fr.h[0, 0, :, 0])
    want = (abs(a1) + abs(a2)) / abs(abs(a1) - abs(a2))
    assert mag.max() / mag.min() == pytest.approx(want, rel=1e-6)


def test_ofdm_linearity_and_oracle(P, golden):
    # T/test_channel.py:96-108: power-of-two scaling is bitwise, complex scaling 1e-13
    rng = np.random.RandomState(3)
    a = rng.randn(3) + 1j * rng.randn(3)
    tau = np.abs(rng.randn(3)) * 1e-7
    h1 = P.frequency_response(_cir(P, a, tau), 32, 30e3).h
    h2 = P.frequency_response(_cir(P, 2.0 * a, tau), 32, 30e3).h
    assert np.array_equal(h2, 2.0 * h1)
    s = 2.5 - 1.25j
    h3 = P.frequency_response(_cir(P, s * a, tau), 32, 30e3).h
    assert np.allclose(h3, s * h1, rtol=1e-13, atol=0)
    # a device CIR of the golden canyon vs the oracle's response of the reference CIR
    g = golden("canyon")
    sc = golden_scene(g)
    bvh = P.build(sc)
    ps = P.compute_paths(sc, bvh, int(g["max_depth"]), method=str(g["method"]),
                         num_rays=int(g["num_rays"]))
    cir = P.build_cir(P.compute_gains(sc, bvh, ps))
    fr = P.frequency_response(cir, 32, 30e3)
    h, f = O.frequency_response(g["cir_a"], g["cir_tau"], 32, 30e3)
    assert np.allclose(fr.h, h, rtol=1e-9, atol=1e-20)
    assert np.array_equal(fr.frequencies, f)
