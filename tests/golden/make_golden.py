"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (the reference is importable there, not on the GPU
box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture records the reference's outputs on seeded inputs produced by
this repo's generators (paper_1308_5467_b200/workloads.py), plus a SHA-256
of the matrix arrays so a drifting generator is caught.  The oracle is pinned
against these files by tests/test_oracle_golden.py and the CUDA path by the
GPU parity tests.
"""

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import scipy  # noqa: E402
import specdens  # noqa: E402
from specdens import (  # noqa: E402
    ProbeVectorSource,
    SparseSymmetricMatrix,
    apply_spectral_map,
    compute_chebyshev_moments,
    compute_legendre_moments,
    delta_chebyshev_dos,
    estimate_dos,
    evaluate_kpml_dos,
    spectroscopic_dos,
    evaluate_kpm_dos,
    lanczos_dos,
    lanczos_factorize,
    moments_to_coefficients,
    moments_via_product_formula,
)
from specdens.density import SpectralInterval, interval_grid, unit_grid  # noqa: E402

from paper_1308_5467_b200 import workloads as W  # noqa: E402


class Shifted:
    """A probe source whose probe i is the reference source's probe start+i."""

    def __init__(self, src, start):
        self.src, self.start, self.dim = src, start, src.dim

    def draw(self, i):
        return self.src.draw(self.start + i)


def csr_digest(csr):
    h = hashlib.sha256()
    for a in (csr.indptr.astype(np.int64), csr.indices.astype(np.int64), csr.data.astype(np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ref_matrix(op):
    return SparseSymmetricMatrix(csr=op.csr)


def kpm_case(name, op, kind, n_vec, degree, n_pts, per_probe=2):
    t0 = time.time()
    mat = ref_matrix(op)
    lb, ub = W.gershgorin_interval(op).lambda_lb, W.gershgorin_interval(op).lambda_ub
    iv = SpectralInterval(lb, ub)
    src = ProbeVectorSource(kind, seed=0, dim=mat.dim)
    mapped = apply_spectral_map(mat, iv)
    direct = compute_chebyshev_moments(mapped, degree, src, n_vec)
    product = moments_via_product_formula(mapped, degree, src, n_vec)
    grid = unit_grid(n_pts)
    dos_d = evaluate_kpm_dos(moments_to_coefficients(direct, "jackson"), iv, grid)
    dos_p = evaluate_kpm_dos(moments_to_coefficients(product, "jackson"), iv, grid)
    pp = np.array([compute_chebyshev_moments(mapped, degree, Shifted(src, l), 1).zeta for l in range(per_probe)])
    out = dict(
        kind=kind, n_vec=n_vec, degree=degree, n_pts=n_pts, lb=lb, ub=ub,
        zeta_direct=direct.zeta, zeta_product=product.zeta, per_probe_direct=pp,
        values_direct=dos_d.values, density_direct=dos_d.density, lambda_grid=dos_d.lambda_grid,
        values_product=dos_p.values, density_product=dos_p.density,
        matrix_sha256=csr_digest(mat.csr), n=mat.dim, nnz=mat.csr.nnz,
    )
    est = estimate_dos(mat, iv, "kpm-jackson", degree, src, n_vec, grid_points=n_pts)
    out["estimate_density"] = est.density
    out["estimate_matvec_count"] = est.params["matvec_count"]
    est_p = estimate_dos(mat, iv, "kpm-jackson", degree, src, n_vec, grid_points=n_pts, product_formula=True)
    out["estimate_density_product"] = est_p.density
    out["estimate_matvec_count_product"] = est_p.params["matvec_count"]
    print(f"{name}: n={mat.dim} nnz={mat.csr.nnz} {time.time() - t0:.1f}s", flush=True)
    return out


def lanczos_case(name, op, kind, n_vec, steps, sigma, n_pts):
    t0 = time.time()
    mat = ref_matrix(op)
    g = W.gershgorin_interval(op)
    iv = SpectralInterval(g.lambda_lb, g.lambda_ub)
    src = ProbeVectorSource(kind, seed=0, dim=mat.dim)
    grid = interval_grid(iv, n_pts)
    est = lanczos_dos(mat, iv, steps, src, n_vec, sigma, grid)
    alphas, betas, bnext = [], [], []
    for l in range(min(n_vec, 2)):
        f = lanczos_factorize(mat, src.draw(l), steps)
        alphas.append(f.alpha)
        betas.append(f.beta)
        bnext.append(f.beta_next)
    est2 = estimate_dos(mat, iv, "lanczos", steps, src, n_vec, sigma=sigma, grid_points=n_pts)
    print(f"{name}: n={mat.dim} {time.time() - t0:.1f}s", flush=True)
    return dict(
        kind=kind, n_vec=n_vec, steps=steps, sigma=sigma, n_pts=n_pts, lb=iv.lambda_lb, ub=iv.lambda_ub,
        grid=grid, density=est.density, ritz_nodes=est.params["ritz_nodes"],
        ritz_weights=est.params["ritz_weights"], alpha=np.array(alphas), beta=np.array(betas),
        beta_next=np.array(bnext), estimate_density=est2.density,
        estimate_matvec_count=est2.params["matvec_count"], matrix_sha256=csr_digest(mat.csr), n=mat.dim,
    )


def variants_case(name, op, kind, n_vec, degree, n_pts):
    """Moment-sharing variants: Legendre moments + KPML, spectroscopic, delta-Chebyshev."""
    t0 = time.time()
    mat = ref_matrix(op)
    g = W.gershgorin_interval(op)
    iv = SpectralInterval(g.lambda_lb, g.lambda_ub)
    src = ProbeVectorSource(kind, seed=0, dim=mat.dim)
    mapped = apply_spectral_map(mat, iv)
    grid = unit_grid(n_pts)
    leg = compute_legendre_moments(mapped, degree, src, n_vec)
    kpml = evaluate_kpml_dos(leg, iv, grid)
    cheb = compute_chebyshev_moments(mapped, degree, src, n_vec)
    spec = spectroscopic_dos(cheb, iv, grid)
    rng = np.random.default_rng(7)
    degrees = rng.integers(0, degree + 1, n_pts)
    delta = delta_chebyshev_dos(cheb, iv, grid, degrees=degrees)
    out = dict(kind=kind, n_vec=n_vec, degree=degree, n_pts=n_pts, lb=iv.lambda_lb, ub=iv.lambda_ub,
               zeta_legendre=leg.zeta, kpml_values=kpml.values, kpml_density=kpml.density,
               zeta_chebyshev=cheb.zeta, spectroscopic_density=spec.density, delta_degrees=degrees,
               delta_density=delta.density, matrix_sha256=csr_digest(mat.csr), n=mat.dim)
    for method in ("kpml", "spectroscopic", "delta-cheb"):
        est = estimate_dos(mat, iv, method, degree, src, n_vec, grid_points=n_pts)
        out[f"estimate_{method}_density"] = est.density
        out[f"estimate_{method}_matvec_count"] = est.params["matvec_count"]
    from specdens.dgl import compute_dgl_coefficients, evaluate_dgl_dos
    sigma = 0.05 * iv.halfwidth
    dgl = evaluate_dgl_dos(leg, iv, sigma, grid)
    out["dgl_sigma"] = sigma
    out["dgl_density"] = dgl.density
    out["dgl_effective_degree"] = dgl.params["effective_degree"]
    est = estimate_dos(mat, iv, "dgl", degree, src, n_vec, sigma=sigma, grid_points=n_pts)
    out["estimate_dgl_density"] = est.density
    out["estimate_dgl_matvec_count"] = est.params["matvec_count"]
    for i, tc in enumerate((-0.9, -0.3, 0.0, 0.55)):
        co = compute_dgl_coefficients(tc, 0.05, degree)
        out[f"dglcoef{i}_t"] = tc
        out[f"dglcoef{i}_gamma"] = co.gamma
        out[f"dglcoef{i}_psi"] = co.psi
        out[f"dglcoef{i}_effective"] = co.effective_degree
    print(f"{name}: n={mat.dim} {time.time() - t0:.1f}s", flush=True)
    return out


def interval_case(name):
    """estimate_spectral_interval (matrix.py:207-241) + ritz_residual_bounds (lanczos.py:162-167)."""
    from specdens import estimate_spectral_interval
    from specdens.lanczos import ritz_residual_bounds
    from specdens.stochastic import INTERVAL_STREAM

    t0 = time.time()
    rng = np.random.default_rng(11)
    a = rng.standard_normal((20, 20))
    mats = {
        "c1": ref_matrix(W.build_matrix("C1")),
        "c2": ref_matrix(W.build_matrix("C2")),
        "dense20": SparseSymmetricMatrix.from_dense(a + a.T),
        "diag10": SparseSymmetricMatrix.from_dense(np.diag(np.arange(1.0, 11.0))),
        "diag3": SparseSymmetricMatrix.from_dense(np.diag([-3.0, 0.0, 5.0])),
    }
    runs = [("c1", 20, 0.01), ("c1", 40, 0.0), ("c2", 20, 0.01), ("dense20", 20, 0.0), ("dense20", 7, 0.05),
            ("diag10", 10, 0.01), ("diag3", 3, 0.01)]
    out = {}
    for i, (key, steps, margin) in enumerate(runs):
        iv = estimate_spectral_interval(mats[key], lanczos_steps=steps, margin=margin, seed=0)
        src = ProbeVectorSource("gaussian", seed=0, dim=mats[key].dim, stream=INTERVAL_STREAM)
        fact = lanczos_factorize(mats[key], src.draw(0), min(steps, mats[key].dim))
        theta, resid = ritz_residual_bounds(fact)
        out[f"run{i}_matrix"] = key
        out[f"run{i}_steps"] = steps
        out[f"run{i}_margin"] = margin
        out[f"run{i}_lb"] = iv.lambda_lb
        out[f"run{i}_ub"] = iv.lambda_ub
        out[f"run{i}_theta"] = theta
        out[f"run{i}_resid"] = resid
    out["runs"] = len(runs)
    out["dense20"] = a + a.T
    print(f"{name}: {time.time() - t0:.1f}s", flush=True)
    return out


def haydock_case(name, op, kind, n_vec, steps, n_pts, eta):
    """haydock_dos (lanczos.py:263-293) and the resolvent routes (lanczos.py:222-260)."""
    from specdens.lanczos import continued_fraction_resolvent, haydock_dos, tridiagonal_resolvent_first

    t0 = time.time()
    mat = ref_matrix(op)
    g = W.gershgorin_interval(op)
    iv = SpectralInterval(g.lambda_lb, g.lambda_ub)
    src = ProbeVectorSource(kind, seed=0, dim=mat.dim)
    grid = interval_grid(iv, n_pts)
    est = haydock_dos(mat, iv, steps, src, n_vec, eta=eta, grid=grid)
    est_default = haydock_dos(mat, iv, steps, src, n_vec, grid=grid)
    est2 = estimate_dos(mat, iv, "haydock", steps, src, n_vec, eta=eta, grid_points=n_pts)
    fact = lanczos_factorize(mat, src.draw(0), steps)
    z = np.linspace(iv.lambda_lb - 1.0, iv.lambda_ub + 1.0, 300) + 1j * eta
    cf = continued_fraction_resolvent(fact.alpha, fact.beta, z)
    w0, wl = tridiagonal_resolvent_first(fact.alpha, fact.beta, z)
    print(f"{name}: n={mat.dim} {time.time() - t0:.1f}s", flush=True)
    return dict(kind=kind, n_vec=n_vec, steps=steps, n_pts=n_pts, eta=eta, lb=iv.lambda_lb, ub=iv.lambda_ub,
                grid=grid, density=est.density, trunc=est.params["truncation_indicator"],
                density_default_eta=est_default.density, default_eta=est_default.params["eta"],
                trunc_default=est_default.params["truncation_indicator"], estimate_density=est2.density,
                estimate_matvec_count=est2.params["matvec_count"], alpha0=fact.alpha, beta0=fact.beta, z=z, cf=cf,
                w_first=w0, w_last=wl, matrix_sha256=csr_digest(mat.csr), n=mat.dim)


MM_FILES = {
    "tridiag_sym.mtx": "%%MatrixMarket matrix coordinate real symmetric\n3 3 5\n1 1 2.0\n2 1 -1.0\n2 2 2.0\n"
                       "3 2 -1.0\n3 3 2.0\n",
    "dup_sym.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1.5\n1 1 0.5\n2 1 -1.0\n",
    "general_comments.mtx": "%%MatrixMarket matrix coordinate real general\n% a comment\n\n4 4 7\n"
                            "1 1 1e-3\n% inner comment\n1 2 -2.5\n2 1 -2.5\n2 2 4\n3 4 0.125\n"
                            "4 3 0.125\n\n4 4 -7.0E+2\n",
    "integer_upper.mtx": "%%MatrixMarket MATRIX Coordinate INTEGER Symmetric\n3 3 4\n1 1 3\n3 1 -1\n2 2 +5\n"
                         "3 3 2\n",
    "zero.mtx": "%%MatrixMarket matrix coordinate real symmetric\n4 4 0\n",
}


def mm_case(name):
    """load_matrix_market / save_matrix_market (matrix.py:247-331) on small files."""
    from specdens.matrix import generate_modified_laplacian_2d, load_matrix_market, save_matrix_market

    d = os.path.join(HERE, "mm")
    os.makedirs(d, exist_ok=True)
    for fname, text in MM_FILES.items():
        with open(os.path.join(d, fname), "w", encoding="ascii") as fh:
            fh.write(text)
    save_matrix_market(generate_modified_laplacian_2d(20, 15), os.path.join(d, "lap20x15.mtx"))
    out = {}
    for fname in sorted(os.listdir(d)):
        mat = load_matrix_market(os.path.join(d, fname))
        key = fname.replace(".mtx", "")
        out[f"{key}_indptr"] = mat.csr.indptr.astype(np.int64)
        out[f"{key}_indices"] = mat.csr.indices.astype(np.int64)
        out[f"{key}_data"] = mat.csr.data
        out[f"{key}_symmetric_storage"] = mat.symmetric_storage
    out["files"] = np.array(sorted(os.listdir(d)))
    print(f"{name}: {len(out['files'])} files", flush=True)
    return out


def main():
    meta = dict(numpy=np.__version__, scipy=scipy.__version__, specdens=specdens.__version__,
                python=sys.version.split()[0])
    cases = {
        "c1_kpm": lambda: kpm_case("c1_kpm", W.build_matrix("C1"), "gaussian", 20, 100, 1000),
        "c2_subset": lambda: kpm_case("c2_subset", W.build_matrix("C2"), "rademacher", 2, 500, 2000),
        "c3_small": lambda: kpm_case("c3_small", W.dft_like(20000), "gaussian", 4, 200, 2000),
        "c5_small": lambda: kpm_case("c5_small", W.stencil27_3d(24), "rademacher", 2, 200, 2000),
        "c4_subset": lambda: lanczos_case("c4_subset", W.build_matrix("C4"), "gaussian", 4, 100, 0.01, 2000),
        "lanczos_small": lambda: lanczos_case("lanczos_small", W.anderson_3d(8), "gaussian", 6, 40, 0.05, 400),
        "haydock_small": lambda: haydock_case("haydock_small", W.anderson_3d(8), "gaussian", 6, 40, 400, 0.05),
        "haydock_c4": lambda: haydock_case("haydock_c4", W.build_matrix("C4"), "gaussian", 4, 100, 2000, 0.01),
        "interval": lambda: interval_case("interval"),
        "matrix_market": lambda: mm_case("matrix_market"),
        "variants_c1": lambda: variants_case("variants_c1", W.build_matrix("C1"), "gaussian", 20, 100, 1000),
        "variants_c5small": lambda: variants_case("variants_c5small", W.stencil27_3d(24), "rademacher", 32, 60,
                                                  500),
    }
    only = sys.argv[1:]
    for name, fn in cases.items():
        if only and name not in only:
            continue
        data = fn()
        data.update({f"meta_{k}": v for k, v in meta.items()})
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **data)


if __name__ == "__main__":
    main()
