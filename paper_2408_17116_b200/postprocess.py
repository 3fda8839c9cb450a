"""Far field and bistatic RCS from a solution vector.
Restates postprocess.py:30-233 (density_grids, _patch_tables native branch,
far_field, rcs_cut): the O(N) quadrature tables are formed on the host, the
O(angles x N) phase-weighted radiation sums run on the device
(cbie_far_field_sums, csrc/farfield.cu)."""

from __future__ import annotations

import numpy as np

from . import _ffi, geometry as geo


def _fejer_weights(n):
    th = (2.0 * np.arange(n) + 1.0) * np.pi / (2.0 * n)
    w = np.ones(n)
    for m in range(1, n // 2 + 1):
        w -= 2.0 * np.cos(2 * m * th) / (4 * m * m - 1)
    return (2.0 / n) * w


def _node_diff(n):
    x = geo.fejer_nodes(n)
    S = geo._vander(x, n)
    return S @ geo._dcoef(n) @ geo._analysis(n)


def radiation_tables(gen, solution):
    """pos, w (a_u F^u + a_v F^v), w div F per node; (M tables for Muller)."""
    C = gen.C
    nu, nv = gen.nu, gen.nv
    npatch = len(gen.patches)
    wgt = (_fejer_weights(nv)[:, None] * _fejer_weights(nu)[None, :]).ravel()
    Du, Dv = _node_diff(nu), _node_diff(nv)
    F = solution.reshape(npatch, nv * nu, C)
    au = gen.a_u.reshape(npatch, nv * nu, 3)
    av = gen.a_v.reshape(npatch, nv * nu, 3)
    out = []
    for cu, cv in ((0, 1), (2, 3))[: C // 2]:
        vec = wgt[None, :, None] * (F[:, :, cu, None] * au + F[:, :, cv, None] * av)
        gu = F[:, :, cu].reshape(npatch, nv, nu)          # [patch][k][l]
        gv = F[:, :, cv].reshape(npatch, nv, nu)
        du = np.einsum("pkl,ml->pkm", gu, Du).reshape(npatch, -1)
        dv = np.einsum("pkl,nk->pnl", gv, Dv).reshape(npatch, -1)
        out.append((vec.reshape(-1, 3), (wgt[None, :] * (du + dv)).reshape(-1)))
    return gen.pos, out


def far_field(problem, gen, solution, theta, phi):
    med = problem.spec.outer
    k, omega = med.k, med.omega
    if abs(np.imag(k)) > 0.0:
        raise ValueError("far field: lossy exterior medium (complex k) is not supported")
    pos, tabs = radiation_tables(gen, solution)
    rhat = np.ascontiguousarray(
        np.stack([np.sin(theta) * np.cos(phi), np.sin(theta) * np.sin(phi), np.cos(theta)], 1))
    cols = [tabs[0][0], tabs[0][1][:, None]]
    if len(tabs) > 1:
        cols.append(tabs[1][0])
    tab = np.ascontiguousarray(np.concatenate(cols, axis=1).astype(complex))
    sums = np.empty((rhat.shape[0], tab.shape[1]), complex)
    gen.dev.check(gen.dev.lib.cbie_far_field_sums(gen.dev.h, _ffi.ptr(tab), int(tab.shape[1]), _ffi.ptr(rhat),
                                                  int(rhat.shape[0]), float(np.real(k)), _ffi.ptr(sums)))
    Jhat, Jdiv = sums[:, 0:3], sums[:, 3]
    F = -(1.0 / (4 * np.pi)) * (1j * omega * med.mu * Jhat + (k / (omega * med.eps)) * rhat * Jdiv[:, None])
    if len(tabs) > 1:
        F = F + (1.0 / (4 * np.pi)) * 1j * k * np.cross(rhat, sums[:, 4:7])
    return F - rhat * np.sum(F * rhat, axis=1)[:, None], rhat


def rcs_cut(problem, gen, solution, phi_deg, theta_deg):
    """sigma (m^2) and sigma (dBsm) over theta at fixed phi (postprocess.py:215-233)."""
    theta = np.deg2rad(np.asarray(theta_deg, float))
    phi = np.full_like(theta, np.deg2rad(phi_deg))
    F, _ = far_field(problem, gen, solution, theta, phi)
    that = np.stack([np.cos(theta) * np.cos(phi), np.cos(theta) * np.sin(phi), -np.sin(theta)], 1)
    phat = np.stack([-np.sin(phi), np.cos(phi), np.zeros_like(phi)], 1)
    et = np.sum(F * that, axis=1)
    ep = np.sum(F * phat, axis=1)
    sigma = 4 * np.pi * (np.abs(et) ** 2 + np.abs(ep) ** 2) / problem.excitation.amplitude ** 2
    return sigma, 10.0 * np.log10(np.maximum(sigma, 1e-300))


def surface_current_vectors(gen, solution):
    """Physical J (and M for Muller) at every node, (N_points, 3) each
    (postprocess.py:45-62): J = (x_u a_u + x_v a_v) / sqrt(g) with the device frames."""
    C = gen.C
    F = np.asarray(solution).reshape(-1, C)
    J = (F[:, 0, None] * gen.a_u + F[:, 1, None] * gen.a_v) / gen.sqrt_g[:, None]
    M = (F[:, 2, None] * gen.a_u + F[:, 3, None] * gen.a_v) / gen.sqrt_g[:, None] if C == 4 else None
    return J, M


def current_error(gen, solution, points_idx, J_ref, w):
    """Weighted relative L2 distance of the surface current to a reference current J_ref
    at the node indices points_idx, weights w = node weight x sqrt(g) -- the
    current_error_weighted of postprocess.mie_comparison (postprocess.py:275-314)."""
    J, _ = surface_current_vectors(gen, solution)
    d2 = np.sum(np.abs(J[points_idx] - J_ref) ** 2, axis=1)
    r2 = np.sum(np.abs(J_ref) ** 2, axis=1)
    return float(np.sqrt((w @ d2) / (w @ r2)))
