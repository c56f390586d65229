"""Golden fixtures for the trace estimator and the heat-capacity functional, made by
running the REFERENCE itself:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_extras.py

tests/test_gpu_extras.py replays them on the GPU path.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from specdens import (  # noqa: E402
    ProbeVectorSource,
    RegularizationKernel,
    RitzQuadrature,
    SparseSymmetricMatrix,
    default_temperatures,
    dense_eigensolve,
    estimate_trace_quadratic,
    exact_regularized_dos,
    generate_modified_laplacian_2d,
    heat_capacity,
    interval_grid,
    spectrum_interval,
)

from paper_1308_5467_b200 import workloads as W  # noqa: E402


def main():
    out = {}
    lap = generate_modified_laplacian_2d(100, 100, bumps=())
    t = estimate_trace_quadratic(lap, ProbeVectorSource("gaussian", seed=0, dim=lap.dim), 50)
    out["trace/c1"] = [t.value, t.n_samples, t.sample_variance]
    op = SparseSymmetricMatrix(csr=W.anderson_3d(8).csr)
    t = estimate_trace_quadratic(op, ProbeVectorSource("rademacher", seed=1, dim=op.dim), 20)
    out["trace/and8"] = [t.value, t.n_samples, t.sample_variance]

    small = generate_modified_laplacian_2d(10, 5)
    spec = dense_eigensolve(small)
    temps = default_temperatures()
    out["heat/temps"] = temps
    out["heat/eigs"] = spec.eigenvalues
    out["heat/exact"] = heat_capacity(spec, temps)
    iv = spectrum_interval(spec, margin=0.05)
    grid = interval_grid(iv, 800)
    est = exact_regularized_dos(spec, RegularizationKernel("gaussian", 0.2), grid, iv)
    out["heat/grid"] = grid
    out["heat/density"] = est.density
    out["heat/interval"] = [iv.lambda_lb, iv.lambda_ub]
    out["heat/estimate"] = heat_capacity(est, temps)
    rng = np.random.default_rng(4)
    theta = np.sort(rng.uniform(0.0, 8.0, 60))
    tau = rng.uniform(0.0, 1.0, 60)
    tau /= tau.sum()
    out["heat/theta"] = theta
    out["heat/tau"] = tau
    out["heat/ritz"] = heat_capacity(RitzQuadrature(theta=theta, tau_sq=tau), temps, normalize=False)
    np.savez_compressed(os.path.join(HERE, "extras.npz"), **out)


if __name__ == "__main__":
    main()
