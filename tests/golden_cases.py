"""The golden fixtures (tests/golden/*.npz, frozen from the live reference by
tests/golden/make_golden.py) and how to rebuild each case's kernel and target
for the oracle (oracle/) and for the device engine (paper_2503_17405_b200)."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


# name -> (variants, kernel spec, target spec)
CASES = {
    "drmh_mog10": (("plain", "bundled", "amortized", "standard"), ("drmh", 100, 0.1), ("mog", 10, 0.9, (-3.0, 0.0, 3.0))),
    "drmh_funnel10": (("plain", "bundled", "standard"), ("drmh", 100, 0.1), ("funnel", 10)),
    "drmh_std1": (("plain", "bundled", "standard"), ("drmh", 100, 0.1), ("gauss", np.zeros(1), np.eye(1))),
    "drmh_gauss3": (("plain", "bundled", "standard"), ("drmh", 20, 0.7),
                    ("gauss", np.array([0.5, -1.0, 2.0]),
                     np.array([[1.0, 0, 0], [0.3, 0.8, 0], [-0.2, 0.1, 0.5]]))),
    "ess_conj100": (("plain", "bundled", "amortized", "standard"), ("ess",), ("conjugate", 100)),
    "ess_conj2": (("plain", "bundled", "standard"), ("ess",), ("conjugate", 2)),
    "ess_gpc64": (("amortized", "bundled", "standard"), ("ess",), ("gpc", 64)),
    "nuts_corr100": (("plain", "bundled", "standard"), ("nuts", 0.05, 10, 1000.0), ("equicorr", 100, 0.99)),
    "nuts_mog10": (("plain", "bundled", "standard"), ("nuts", 0.2, 6, 1000.0), ("mog", 10, 0.9, (-3.0, 0.0, 3.0))),
    "nuts_funnel5": (("plain", "bundled", "standard"), ("nuts", 0.3, 5, 50.0), ("funnel", 5)),
    "nuts_std2": (("plain", "bundled", "standard"), ("nuts", 0.9, 4, 1000.0), ("gauss", np.zeros(2), np.eye(2))),
    "nuts_logreg512x16": (("plain", "bundled", "standard"), ("nuts", 0.1, 8, 1000.0), ("logreg",)),
    "drmh_split_std1": (("plain", "bundled", "standard"), ("drmh-split", 50, 0.4), ("gauss", np.zeros(1), np.eye(1))),
    "drmh_split_mog10": (("plain", "bundled", "standard"), ("drmh-split", 100, 0.1), ("mog", 10, 0.9, (-3.0, 0.0, 3.0))),
    "slice_std1": (("plain", "bundled", "amortized", "standard"), ("slice", 1.0, 32), ("gauss", np.zeros(1), np.eye(1))),
    "slice_narrow": (("plain", "bundled", "standard"), ("slice", 0.2, 50), ("gauss", np.array([1.5]), np.array([[2.0]]))),
    "slice_cap": (("plain", "bundled", "standard"), ("slice", 0.05, 3), ("gauss", np.zeros(1), np.eye(1))),
    "slice_box": (("plain", "bundled", "standard"), ("slice", 10.0, 8), ("box", 1, 0.0, 1.0)),
    "ess_gp50": (("amortized", "bundled", "standard"), ("ess",), ("gphyper", "ess_gp50")),
    "drmh_gp50": (("plain", "bundled", "standard"), ("drmh", 20, 0.2), ("gphyper", "drmh_gp50")),
    "nuts_gp50": (("plain", "bundled", "standard"), ("nuts", 0.1, 6, 1000.0), ("gphyper", "nuts_gp50")),
}

# sample tolerance per case (relative, |a-b| <= tol max(1, |b|)): 1e-12 by default; the
# GP cases factor a 50 x 50 kernel matrix whose LAPACK (OpenBLAS) operation order is
# not restated, and cond(K) ~ 1e3 amplifies the last-ulp differences
SAMPLE_TOL = {"ess_gp50": 1e-9, "drmh_gp50": 1e-9, "nuts_gp50": 1e-9}


def sample_tol(name):
    return SAMPLE_TOL.get(name, 1e-12)

# cases the oracle does not restate (checked against the goldens on the device only)
DEVICE_ONLY = {"drmh_split_std1", "drmh_split_mog10"}


def x0_of(g):
    """The case's start point (None: the default zeros)."""
    return g["x0"] if "x0" in g.files else None


def oracle_kernel(spec):
    from oracle import oracle as O
    if spec[0] == "slice":
        return O.slice_(spec[1], spec[2])
    if spec[0] == "drmh":
        return O.drmh(spec[1], spec[2])
    if spec[0] == "ess":
        return O.elliptical()
    return O.nuts(spec[1], spec[2], spec[3])


def oracle_target(spec):
    from oracle import oracle as O
    kind = spec[0]
    if kind == "mog":
        return O.mog(spec[1], spec[2], list(spec[3]))
    if kind == "funnel":
        return O.funnel(spec[1])
    if kind == "box":
        return O.box(spec[1], spec[2], spec[3])
    if kind == "gphyper":
        g = load(spec[1])
        return O.gp_hyper(g["X"], g["y"])
    if kind == "gauss":
        return O.gaussian(spec[1], spec[2])
    if kind == "equicorr":
        return O.gaussian(np.zeros(spec[1]), np.linalg.cholesky(O.equicorrelated_covariance(spec[1], spec[2])))
    if kind == "conjugate":
        return O.conjugate(spec[1])
    if kind == "gpc":
        g = load("ess_gpc64")
        return O.logistic_fspace(g["L"], g["y"])
    if kind == "logreg":
        g = load("nuts_logreg512x16")
        return O.logreg(g["X"], g["y"])
    raise KeyError(kind)


def device_kernel(spec):
    import paper_2503_17405_b200 as fm
    if spec[0] == "drmh-split":
        return fm.drmh_kernel(spec[1], spec[2], split_body=True)
    if spec[0] == "slice":
        return fm.slice_kernel(spec[1], spec[2])
    if spec[0] == "drmh":
        return fm.drmh_kernel(spec[1], spec[2])
    if spec[0] == "ess":
        return fm.elliptical_kernel()
    return fm.nuts_kernel(spec[1], spec[2], spec[3])


def device_target(spec, structure="auto"):
    import paper_2503_17405_b200 as fm
    from paper_2503_17405_b200 import targets as T
    kind = spec[0]
    if kind == "mog":
        return fm.correlated_mog_target(spec[1], spec[2], list(spec[3]))
    if kind == "funnel":
        return fm.funnel_target(spec[1])
    if kind == "box":
        return fm.box_target(spec[1], spec[2], spec[3])
    if kind == "gphyper":
        g = load(spec[1])
        return fm.gp_hyperparameter_target(g["X"], g["y"])
    if kind == "gauss":
        return fm.gaussian_target(spec[1], spec[2], structure=structure)
    if kind == "equicorr":
        return fm.gaussian_target(np.zeros(spec[1]),
                                  np.linalg.cholesky(fm.equicorrelated_covariance(spec[1], spec[2])),
                                  structure=structure)
    if kind == "conjugate":
        return fm.conjugate_target(spec[1])
    if kind == "gpc":
        return T.gp_classification_target(spec[1])
    if kind == "logreg":
        g = load("nuts_logreg512x16")
        return T.logistic_regression_target(g["X"], g["y"])
    raise KeyError(kind)


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0
