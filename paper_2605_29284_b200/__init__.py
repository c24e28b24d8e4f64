"""paper_2605_29284_b200 — B200-native rapid approximate Kriging (arXiv 2605.29284).

Drop-in for the hot path of the reference package ``rapidkrig`` (same names and
signatures, re-exported like reference __init__.py:16-49): rapid grid
prediction and the fast conditional-simulation ensemble built on it.  All
arithmetic runs in ``librapidkrig_b200.so`` (hand-written sm_100a CUDA behind a
C ABI, include/rapidkrig_b200.h); there is no CPU fallback.
"""

from .covariance import CovarianceModel, cov, cov_matrix, matern_phi
from .errors import DomainError, InternalError, NumericError, RapidKrigError
from .exact import KrigingFit, as_device_fit, fit, kriging_se_exact, predict_exact, refit_coefficients
from .gridding import (NODE_SNAP_TOL, Neighborhood, PaddedGrid, build_padded_grid,
                       fill_distance, neighborhood)
from .rapid import (RapidSetup, build_filter_spectrum, build_setup, convolve_filter,
                    neighbor_cov, next_fft_len, predict_rapid)
from .simulate import (RNG_ALGORITHM, Ensemble, conditional_draw, draw_seed,
                       generate_ensemble, sim_obs_local, sim_unconditional_grid)
from . import rapid

__version__ = "0.1.0"

__all__ = [
    "CovarianceModel", "cov", "cov_matrix", "matern_phi",
    "RapidKrigError", "DomainError", "NumericError", "InternalError",
    "KrigingFit", "fit", "refit_coefficients", "predict_exact", "kriging_se_exact", "as_device_fit",
    "PaddedGrid", "Neighborhood", "build_padded_grid", "neighborhood", "fill_distance",
    "NODE_SNAP_TOL",
    "RapidSetup", "build_setup", "predict_rapid", "next_fft_len", "build_filter_spectrum",
    "convolve_filter", "neighbor_cov", "rapid",
    "Ensemble", "RNG_ALGORITHM", "draw_seed", "sim_unconditional_grid", "sim_obs_local",
    "conditional_draw", "generate_ensemble",
]
