"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no covariances, no Toeplitz, no
SVD, no pole extraction). It only draws the inputs of the paper's discrete stochastic
state-space model, Eq. (5) (§2.1):

    x_{h+1} = A x_h + w_h,   y_h = C x_h + v_h

in modal coordinates, plus the generating poles of Eq. (3) so tests can
compare identified poles against the truth. The per-config recipe is SURVEY.md §8(d)
and is restated in DESIGN.md §"Input recipe".
"""
from .records import (CONFIGS, Config, Modes, make_modes, make_record, make_batch_record,
                      exact_poles, config)

__all__ = ["CONFIGS", "Config", "Modes", "make_modes", "make_record", "make_batch_record",
           "exact_poles", "config"]
