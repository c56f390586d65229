"""Golden fixtures for ``run_method_comparison`` made by running the REFERENCE itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_comparison.py

Each case stores the matrix (CSR arrays, built by the reference's own
generator), the interval and spectrum the reference used, and every row the
reference returned (per-rep errors, means, std, masses, MATVEC counts).
tests/test_gpu_comparison.py replays the same call through the GPU path.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import specdens  # noqa: E402
from specdens import (  # noqa: E402
    dense_eigensolve,
    estimate_spectral_interval,
    generate_modified_laplacian_2d,
    run_method_comparison,
)

METHODS = ["kpm", "kpm-jackson", "spectroscopic", "delta-cheb", "kpml", "dgl", "lanczos", "haydock", "cdos", "exact"]

CASES = {
    # the reference's own conftest matrix (50-dim, default bumps), interval and spectrum passed in
    "small_lap": dict(nx=10, ny=5, methods=METHODS, degrees=[16, 8, 30, 8], sigma=0.5, eta=None, n_vec=8, reps=3,
                      seed=0, probe_kind="gaussian", grid_points=512, pass_interval=True),
    # 24-dim: Lanczos steps capped at the dimension; interval and spectrum computed inside
    "tiny_capped": dict(nx=6, ny=4, methods=["kpm", "lanczos", "haydock", "cdos", "dgl", "exact"], degrees=[10, 30],
                        sigma=0.6, eta=0.3, n_vec=5, reps=4, seed=3, probe_kind="rademacher", grid_points=600,
                        pass_interval=False),
    # exhaustive basis probes (sqrt(n) e_l) on a 12-dim matrix: exact traces, Lanczos to full depth
    "basis_full": dict(nx=4, ny=3, methods=["kpm", "kpm-jackson", "lanczos", "cdos", "exact"], degrees=[5, 12],
                       sigma=0.8, eta=None, n_vec=12, reps=2, seed=0, probe_kind="basis", grid_points=400,
                       pass_interval=False),
}


def main():
    out = {}
    for name, c in CASES.items():
        mat = generate_modified_laplacian_2d(c["nx"], c["ny"])
        kwargs = dict(eta=c["eta"], n_vec=c["n_vec"], reps=c["reps"], seed=c["seed"], probe_kind=c["probe_kind"],
                      grid_points=c["grid_points"])
        iv = estimate_spectral_interval(mat, seed=c["seed"])
        spec = dense_eigensolve(mat)
        if c["pass_interval"]:
            kwargs.update(interval=iv, spectrum=spec)
        rows = run_method_comparison(mat, c["methods"], c["degrees"], c["sigma"], **kwargs)
        csr = mat.csr
        p = name + "/"
        out[p + "indptr"] = np.asarray(csr.indptr, dtype=np.int64)
        out[p + "indices"] = np.asarray(csr.indices, dtype=np.int64)
        out[p + "data"] = np.asarray(csr.data, dtype=np.float64)
        out[p + "interval"] = np.array([iv.lambda_lb, iv.lambda_ub])
        out[p + "eigenvalues"] = spec.eigenvalues
        out[p + "methods"] = np.array(c["methods"])
        out[p + "degrees"] = np.array(c["degrees"])
        out[p + "scalars"] = np.array([c["sigma"], np.nan if c["eta"] is None else c["eta"], c["n_vec"], c["reps"],
                                       c["seed"], c["grid_points"], float(c["pass_interval"])])
        out[p + "probe_kind"] = np.array(c["probe_kind"])
        out[p + "row_method"] = np.array([r.method for r in rows])
        out[p + "row_degree"] = np.array([r.degree for r in rows])
        out[p + "row_matvec"] = np.array([r.matvec_count for r in rows])
        out[p + "row_mean"] = np.array([r.error_mean for r in rows])
        out[p + "row_std"] = np.array([r.error_std for r in rows])
        out[p + "row_mass"] = np.array([r.mass_mean for r in rows])
        out[p + "row_errors"] = np.stack([r.errors for r in rows])
        print(name, len(rows), "rows", file=sys.stderr)
    out["specdens_version"] = np.array(getattr(specdens, "__version__", "unknown"))
    np.savez_compressed(os.path.join(HERE, "method_comparison.npz"), **out)


if __name__ == "__main__":
    main()
