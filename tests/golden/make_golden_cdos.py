"""Golden fixtures for CDOS (lanczos.py:296-368) made by running the REFERENCE itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cdos.py

Cases: cdos_refine on a synthetic pooled quadrature with near-duplicate nodes
(merging), the two-node case of pkg/tests/test_lanczos.py:250-259, a
single-point grid (spline derivative), and cdos_dos / estimate_dos('cdos') on
the reference's 50-dim test Laplacian and on an 8^3 Anderson model.
tests/test_gpu_cdos.py replays them on the GPU path.
"""

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from specdens import (  # noqa: E402
    ProbeVectorSource,
    RitzQuadrature,
    SparseSymmetricMatrix,
    SpectralInterval,
    cdos_dos,
    cdos_refine,
    estimate_dos,
    estimate_spectral_interval,
    generate_modified_laplacian_2d,
    interval_grid,
)
import sys  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1308_5467_b200 import workloads as W  # noqa: E402


def main():
    out = {}
    rng = np.random.default_rng(11)
    theta = np.sort(rng.uniform(-2.0, 3.0, 300))
    theta[50:55] = theta[50] + np.arange(5) * 1e-12  # merged cluster
    theta[200] = theta[199]                          # exact duplicate
    tau = rng.uniform(0.1, 1.0, 300)
    tau /= tau.sum()
    iv = SpectralInterval(-2.5, 3.5)
    grid = interval_grid(iv, 700)
    est = cdos_refine(RitzQuadrature(theta=theta, tau_sq=tau), iv, grid=grid)
    out.update({"syn/theta": theta, "syn/tau": tau, "syn/interval": [iv.lambda_lb, iv.lambda_ub], "syn/grid": grid,
                "syn/density": est.density, "syn/nodes": est.params["nodes"],
                "syn/node_weights": est.params["node_weights"]})
    one = np.array([0.37])
    est1 = cdos_refine(RitzQuadrature(theta=theta, tau_sq=tau), iv, grid=one)
    out["syn/density_one_point"] = est1.density
    two = cdos_refine(RitzQuadrature(theta=np.array([0.0, 1.0]), tau_sq=np.array([0.5, 0.5])),
                      SpectralInterval(-0.5, 1.5), grid=interval_grid(SpectralInterval(-0.5, 1.5), 4001))
    out["two/density"] = two.density

    lap = generate_modified_laplacian_2d(10, 5)
    iv = estimate_spectral_interval(lap, seed=0)
    grid = interval_grid(iv, 512)
    est = cdos_dos(lap, iv, 20, ProbeVectorSource("gaussian", seed=3, dim=lap.dim), 8, grid=grid)
    csr = lap.csr
    out.update({"lap/indptr": np.asarray(csr.indptr, np.int64), "lap/indices": np.asarray(csr.indices, np.int64),
                "lap/data": csr.data, "lap/interval": [iv.lambda_lb, iv.lambda_ub], "lap/density": est.density,
                "lap/ritz_nodes": est.params["ritz_nodes"], "lap/ritz_weights": est.params["ritz_weights"]})

    op = W.anderson_3d(8)
    iv = W.gershgorin_interval(op)
    ref = SparseSymmetricMatrix(csr=op.csr)
    est = estimate_dos(ref, iv, "cdos", 30, ProbeVectorSource("rademacher", seed=0, dim=op.dim), 6, grid_points=300)
    out.update({"and/interval": [iv.lambda_lb, iv.lambda_ub], "and/density": est.density,
                "and/lambda_grid": est.lambda_grid, "and/matvec_count": est.params["matvec_count"]})
    np.savez_compressed(os.path.join(HERE, "cdos.npz"), **out)


if __name__ == "__main__":
    main()
