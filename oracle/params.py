"""Parameter rules printed in the paper (used by pins and drivers' planning only).

  Eq. (tlag)  τ = (2 j_b − 1)/f_s                         PAPER.md:352-354 (§3.1.2)
  Eq. (empirical_formula) k̄(T) = max{30 − 0.00156 T; 25} %  PAPER.md:367-371 (§3.1.2)
  sample count k = ceil(k̄ T / 100)   ("512 columns out of 1890")
  Eq. (jb)    j_b = int(10 f_s / (2 f_0))                 PAPER.md:378-382 (§3.1.3)
  Eq. (jb_3D) j_min = int(9 f_s/(2 f_0)), j_max = β j_min
"int" is read as ceiling (reading A-8: reproduces 189, 76, 170, 69; floor gives 188, 75).
The lag grid is j_min : floor((j_max − j_min)/(G − 1)) : j_max (reading A-9), which ends
at 251 for the 10-DOF case ("spanning from 170 to 251").
"""
import math


def time_lag_step(fs: float, f0: float) -> int:
    return math.ceil(10.0 * fs / (2.0 * f0))


def lag_of_step(j_b: int, fs: float) -> float:
    return (2 * j_b - 1) / fs


def lag_grid(fs: float, f0: float, beta: float, count: int):
    j_min = math.ceil(9.0 * fs / (2.0 * f0))
    j_max = math.ceil(beta * j_min)
    step = (j_max - j_min) // (count - 1)
    return list(range(j_min, j_max + 1, step))[:count], j_min, j_max


def min_rank_percent(T: float) -> float:
    return max(30.0 - 0.00156 * T, 25.0)


def sample_count(percent: float, T: int) -> int:
    return min(max(math.ceil(percent * T / 100.0 - 1e-9), 1), T)
