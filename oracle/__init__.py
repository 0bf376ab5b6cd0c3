"""CPU FP64 ORACLE for the RSVD-accelerated CoV-SSI hot path (arXiv 2411.05510).

TEST INFRASTRUCTURE ONLY. Nothing on the product path may import, call, link or execute
anything under oracle/: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs use it. It shares no code with the CUDA path
(paper_2411_05510_b200/) and neither imports the other; both read inputs made by synth/.

Plain, slow, obviously correct numpy/LAPACK implementations, each function citing the
PAPER.md passage it follows (line numbers of /root/reference/PAPER.md, then section /
equation). Where the paper is silent or garbled the reading is SURVEY.md §8(c)'s and is
listed in DESIGN.md §"Readings". Library primitives used as single steps: matmul,
Householder QR (LAPACK dgeqrf via numpy.linalg.qr), SVD (dgesdd), pinv (SVD-based),
eig (dgeev).

Pins (tests/test_oracle_*.py, -m "not gpu"): every function here is checked against
something other than itself (closed forms, the paper's printed values in
tests/golden/, published Philox known-answer vectors, special cases, brute force on
tiny inputs). No function is "parity unpinned".
"""
from .covariance import covariances, covariance_partial_sums
from .toeplitz import toeplitz
from .philox import philox4x32_10, philox_words, gaussian_sketch, uniforms_from_words
from .rsvd import householder_qr, rsvd, full_svd
from .modal import modal_sweep, poles_from_eigs, Pole, OrderCell
from .indicators import mac, mpc, mpd, normalize_shape
from .stab import stab3d, Criteria, HC_DEFAULT, SC_10DOF_3D, SC_BRIDGE_3D
from .params import (time_lag_step, lag_of_step, lag_grid, min_rank_percent,
                     sample_count)
from .cluster import (stable_pole_features, fuzzy_cmeans, fcm_memberships, select_physical,
                      pole_distances, hierarchical_clusters, cluster_3d)
from .track import track_session, success_ratio
from .preprocess import detrend, preprocess, lowpass_sos, filtfilt_zero_state, rate_ratio
from .frame import frame_matrices, discretize, simulate as simulate_frame

__all__ = [
    "covariances", "covariance_partial_sums", "toeplitz", "philox4x32_10", "philox_words",
    "gaussian_sketch", "uniforms_from_words", "householder_qr", "rsvd", "full_svd",
    "modal_sweep", "poles_from_eigs", "Pole", "OrderCell", "mac", "mpc", "mpd",
    "normalize_shape", "stab3d", "Criteria", "HC_DEFAULT", "SC_10DOF_3D", "SC_BRIDGE_3D",
    "time_lag_step", "lag_of_step", "lag_grid", "min_rank_percent", "sample_count",
    "stable_pole_features", "fuzzy_cmeans", "fcm_memberships", "select_physical", "pole_distances",
    "hierarchical_clusters", "cluster_3d", "track_session", "success_ratio",
    "detrend", "preprocess", "lowpass_sos", "filtfilt_zero_state", "rate_ratio",
    "frame_matrices", "discretize", "simulate_frame",
]
