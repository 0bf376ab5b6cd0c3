"""Block-Toeplitz matrix T_{1|j_b}, Eq. (6) (§2.1).

    T = [[R_{j_b},     R_{j_b−1},  ..., R_1      ],
         [R_{j_b+1},   R_{j_b},    ..., R_2      ],
         ...
         [R_{2j_b−1},  R_{2j_b−2}, ..., R_{j_b}  ]]

i.e. block (r, c) = R_{i + r − c}, r, c ∈ [0, i). Written as the plain double loop.
"""
import numpy as np


def toeplitz(R, i: int) -> np.ndarray:
    """R[k-1] = R_k for k = 1..2i−1 (at least). Returns T [l·i][l·i] FP64."""
    R = np.asarray(R, dtype=np.float64)
    l = R.shape[1]
    T = np.empty((l * i, l * i))
    for r in range(i):
        for c in range(i):
            T[r * l:(r + 1) * l, c * l:(c + 1) * l] = R[(i + r - c) - 1]
    return T
