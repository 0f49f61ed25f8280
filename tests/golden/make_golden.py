"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``divuq`` from /root/reference/pkg/src (read-only; nothing is
copied) and writes small ``.npz`` fixtures next to this file.  The GPU box has
no /root/reference, so only the committed fixtures travel; the tests never
import the reference.

Fixture cases follow the reference's own tests (pkg/tests/conftest.py:12-20
``random_model``; test_divergence.py; test_gaussian.py; test_lcp.py;
test_mc.py) plus edge cases: 2x2 and 2xN/Nx2 grids (all-boundary stencils),
anisotropic spacing, zero / subnormal sigma, extreme tails.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF_SRC)
    import divuq  # noqa: E402
    import importlib

    lcp_mod = importlib.import_module("divuq.lcp")

    return divuq, lcp_mod


def random_model(divuq, grid, rng, sigma_range=(0.05, 0.6)):
    n = grid.n_vertices
    return divuq.GaussianVectorField(
        grid,
        rng.normal(0.0, 2.0, n),
        rng.normal(0.0, 2.0, n),
        rng.uniform(*sigma_range, n),
        rng.uniform(*sigma_range, n),
    )


def main():
    divuq, lcp_mod = _ref()
    rng = np.random.default_rng(20240817)  # pkg/tests/conftest.py:9

    # ---- propagate_divergence (divergence.py:48-70) ----------------------
    grids = [
        (2, 2, 1.0, 1.0), (3, 3, 1.0, 1.0), (13, 7, 0.3, 0.9), (17, 23, 0.21, 1.3),
        (2, 9, 0.5, 0.7), (9, 2, 1.7, 0.4), (64, 48, 0.5, 2.0), (120, 90, 0.2, 0.9),
        (33, 65, 1.0, 1.0),
    ]
    prop = {}
    for gi, (nx, ny, dx, dy) in enumerate(grids):
        g = divuq.UniformGrid2(nx, ny, dx, dy)
        m = random_model(divuq, g, rng)
        # sprinkle exact zeros into sigma to exercise the sigma==0 path downstream
        su = m.sigma_u.copy()
        su[:: 7] = 0.0
        m = divuq.GaussianVectorField(g, m.mu_u, m.mu_v, su, m.sigma_v)
        out = divuq.propagate_divergence(m)
        det = divuq.divergence_deterministic(m.mean_field())
        prop[f"g{gi}_grid"] = np.array([nx, ny, dx, dy])
        prop[f"g{gi}_mu_u"] = m.mu_u
        prop[f"g{gi}_mu_v"] = m.mu_v
        prop[f"g{gi}_s_u"] = m.sigma_u
        prop[f"g{gi}_s_v"] = m.sigma_v
        prop[f"g{gi}_out_mu"] = out.mu
        prop[f"g{gi}_out_sigma"] = out.sigma
        prop[f"g{gi}_det"] = det.values
        for t in (0.0, 0.3):
            below, above = lcp_mod._tail_probs(out.mu, out.sigma, t)
            prop[f"g{gi}_t{t}_above"] = above
            below_n, _ = lcp_mod._tail_probs(out.mu, out.sigma, -t)
            prop[f"g{gi}_t{t}_below_neg"] = below_n
    prop["n_grids"] = np.array(len(grids))
    np.savez_compressed(os.path.join(OUT, "propagate2d.npz"), **prop)

    # ---- lcp (lcp.py:71-100): per-cell crossing probability --------------
    lc = {}
    for gi, (nx, ny, iso) in enumerate([(9, 6, 0.2), (5, 4, -0.1), (33, 17, 0.0), (2, 2, 0.5)]):
        g = divuq.UniformGrid2(nx, ny)
        mu = rng.normal(size=g.n_vertices)
        sg = rng.uniform(0.01, 1.0, g.n_vertices)
        sg[::5] = 0.0
        fld = divuq.GaussianScalarField(g, mu, sg)
        lc[f"l{gi}_grid"] = np.array([nx, ny, iso])
        lc[f"l{gi}_mu"], lc[f"l{gi}_sigma"] = mu, sg
        lc[f"l{gi}_lcp"] = divuq.lcp(fld, iso).probabilities
    cm = rng.normal(0.0, 1.0, (300, 4))
    cs = rng.uniform(0.05, 1.5, (300, 4))
    cs[::7, 2] = 0.0
    lc["cells_mu"], lc["cells_sigma"] = cm, cs
    lc["cells_lcp"] = divuq.cell_crossing_probability(cm, cs, 0.3)
    lc["n_grids"] = np.array(4)
    np.savez_compressed(os.path.join(OUT, "lcp.npz"), **lc)

    # ---- Fig. 1 golden (test_divergence.py:16-21) -------------------------
    fig1 = ((5.98, 0.96), (6.40, 0.38), (6.50, 0.94), (4.30, 0.65))
    mu, sd = divuq.stencil_distribution(fig1, (1.0, 1.0))
    np.savez_compressed(
        os.path.join(OUT, "fig1.npz"),
        neighbors=np.array(fig1), mu=np.array(mu), sigma=np.array(sd),
    )

    # ---- _tail_probs (lcp.py:48-68): probability-map edge cases ----------
    n = 4000
    mu_t = np.concatenate([
        rng.normal(0.0, 3.0, n), rng.uniform(-40, 40, n), [0.0, 0.3, -0.3, 1e8, -1e8, 5.0, -5.0],
    ])
    sg_t = np.concatenate([
        rng.uniform(0.01, 2.0, n), rng.uniform(0.5, 1.5, n), [0.0, 0.0, 0.0, 1e-8, 1e-8, 1e-310, 1e-310],
    ])
    sg_t[::50] = 0.0
    tails = {"mu": mu_t, "sigma": sg_t}
    for t in (0.0, 0.1, 0.3, -0.7):
        b, a = lcp_mod._tail_probs(mu_t, sg_t, t)
        tails[f"t{t}_below"] = b
        tails[f"t{t}_above"] = a
    np.savez_compressed(os.path.join(OUT, "tail_probs.npz"), **tails)

    # ---- fit_gaussian (gaussian.py:35-45) ---------------------------------
    fits = {}
    cases = [(2, 4, 3), (4, 5, 4), (7, 6, 5), (20, 16, 12), (33, 8, 8)]
    for ci, (m_members, nx, ny) in enumerate(cases):
        g = divuq.UniformGrid2(nx, ny)
        members = tuple(
            divuq.VectorField2(
                g,
                rng.normal(5.0, 0.5, g.n_vertices).astype(np.float32).astype(np.float64),
                rng.normal(-1.0, 2.0, g.n_vertices),
            )
            for _ in range(m_members)
        )
        if ci == 1:  # degenerate: four identical members (test_gaussian.py:30-40)
            members = (members[0],) * 4
        model = divuq.fit_gaussian(divuq.Ensemble2(g, members))
        fits[f"c{ci}_shape"] = np.array([m_members, nx, ny])
        fits[f"c{ci}_members"] = np.stack([np.stack([mm.u, mm.v]) for mm in members])
        fits[f"c{ci}_mu_u"] = model.mu_u
        fits[f"c{ci}_mu_v"] = model.mu_v
        fits[f"c{ci}_s_u"] = model.sigma_u
        fits[f"c{ci}_s_v"] = model.sigma_v
    # a generate_synthetic ensemble, the reference's own member recipe
    g = divuq.UniformGrid2(24, 20)
    ens = divuq.generate_synthetic("source-sink", g, 20, 0.3, seed=55)
    model = divuq.fit_gaussian(ens)
    fits["syn_members"] = np.stack([np.stack([mm.u, mm.v]) for mm in ens.members])
    fits["syn_mu_u"], fits["syn_mu_v"] = model.mu_u, model.mu_v
    fits["syn_s_u"], fits["syn_s_v"] = model.sigma_u, model.sigma_v
    an = divuq.propagate_divergence(model)
    fits["syn_div_mu"], fits["syn_div_sigma"] = an.mu, an.sigma
    fits["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "fit_gaussian.npz"), **fits)

    # ---- mc_divergence (mc.py:94-117): reference estimates ----------------
    g = divuq.UniformGrid2(16, 12, 0.5, 0.75)
    m = random_model(divuq, g, rng)
    est = divuq.mc_divergence(m, divuq.McConfig(4000, seed=5))
    an = divuq.propagate_divergence(m)
    np.savez_compressed(
        os.path.join(OUT, "mc_ref.npz"),
        grid=np.array([16, 12, 0.5, 0.75]), mu_u=m.mu_u, mu_v=m.mu_v, s_u=m.sigma_u,
        s_v=m.sigma_v, n_samples=np.array(4000), mean=est.mean, std=est.std,
        an_mu=an.mu, an_sigma=an.sigma,
    )
    # ---- gradient prologue (gaussian.py:48-66) -- appended last so the
    # earlier fixtures' random draws are unchanged
    gr = {}
    g = divuq.UniformGrid2(19, 13, 0.3, 0.7)
    members = tuple(
        divuq.VectorField2(g, rng.normal(size=g.n_vertices), rng.normal(size=g.n_vertices))
        for _ in range(4)
    )
    out = divuq.gradient_ensemble(divuq.Ensemble2(g, members))
    gr["members"] = np.stack([np.stack([m.u, m.v]) for m in members])
    gr["out"] = np.stack([np.stack([m.u, m.v]) for m in out.members])
    gr["vmag0"] = divuq.velocity_magnitude(members[0]).values
    gr["grid"] = np.array([19, 13, 0.3, 0.7])
    np.savez_compressed(os.path.join(OUT, "gradient.npz"), **gr)

    # ---- DIVUQ1 container (io.py:43-55): files written by the reference's
    # own writer, for byte-identity of ours and parsing of theirs
    from divuq import io as ref_io

    for name, (nx, ny, dx, dy, m) in {
        "ens_a": (6, 5, 0.5, 2.0, 4), "ens_b": (7, 3, 0.1, 1e-3, 3),
        "ens_c": (3, 4, 123456.789, 3.0e-7, 2), "ens_d": (2, 2, 1e16, 0.3333333333333333, 5),
    }.items():
        g = divuq.UniformGrid2(nx, ny, dx, dy)
        members = tuple(
            divuq.VectorField2(g, rng.normal(size=g.n_vertices), rng.normal(size=g.n_vertices))
            for _ in range(m)
        )
        ref_io.write_members(g, members, os.path.join(OUT, f"divuq1_{name}.duq"))

    # ---- CLI routing (cli.py:58-107,152-155): the reference CLI's own outputs
    # for the wind-scale pipeline of pkg/tests/test_cli.py:14-40
    from divuq.cli import cli_main

    def p(name):
        return os.path.join(OUT, f"cli_{name}")

    ens = divuq.generate_synthetic("source-sink", divuq.UniformGrid2(24, 24), 15, 0.3, seed=7)
    ref_io.write_ensemble(ens, p("wind.duq"))
    steps = [
        ["fit", "--in", p("wind.duq"), "--out-mu", p("mu.duq"), "--out-sigma", p("sg.duq")],
        ["div", "--in-mu", p("mu.duq"), "--in-sigma", p("sg.duq"), "--out-mu", p("dmu.duq"),
         "--out-sigma", p("dsg.duq")],
        ["lcp", "--in-mu", p("dmu.duq"), "--in-sigma", p("dsg.duq"), "--iso", "-2.525",
         "--out", p("lcp.csv")],
        ["gradmag", "--in", p("wind.duq"), "--out", p("gm.duq")],
    ]
    for argv in steps:
        assert cli_main(argv) == 0, argv
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
