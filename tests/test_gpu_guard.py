"""Out-of-bounds write and input-integrity guards (-m gpu), in place of compute-sanitizer (closed on
this GPU pool): every output array and workspace handed to the C ABI is the interior of a larger
allocation whose margins hold a byte pattern; after the calls the margins must be untouched and
the inputs bit-identical. Covers covariances (three modes), Toeplitz, both RSVD entry points
(k <= 224, k > 224 and k > 512 kernels), the modal sweep, stab3d, the NEXT-2 clustering and
tracking and the NEXT-4 preprocessing and frame generator, at ragged sizes."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MARGIN = 4096          # bytes on each side
PAT = 0xA5


@pytest.fixture(scope="module")
def api():
    from paper_2411_05510_b200 import api, build
    build.build()
    return api


class Guard:
    def __init__(self):
        self.bufs = []

    def take(self, shape, dtype=torch.float64, fill=None):
        n = int(np.prod(shape)) if shape else 1
        es = torch.empty((), dtype=dtype).element_size()
        raw = torch.full((2 * MARGIN + n * es,), PAT, dtype=torch.uint8, device="cuda")
        t = raw[MARGIN: MARGIN + n * es].view(dtype).view(*shape)
        if fill is not None:
            t.copy_(fill)
        self.bufs.append(raw)
        return t

    def ws(self, nbytes):
        t = self.take((max(int(nbytes), 256),), torch.uint8)
        t.zero_()
        return t

    def check(self):
        torch.cuda.synchronize()
        for raw in self.bufs:
            assert torch.all(raw[:MARGIN] == PAT) and torch.all(raw[-MARGIN:] == PAT), "write outside a buffer"


def _table(api, g, n_min, n_max, n_step, l):
    O = (n_max - n_min) // n_step + 1
    cap = n_max // 2
    z = lambda *s, dt=torch.float64: g.take(s, dt, fill=torch.zeros(s, dtype=dt))
    return api.PoleTable(n_min, n_step, l, cap, z(O, dt=torch.int32), z(O, cap), z(O, cap), z(O, cap), z(O, cap),
                         z(O, cap), z(O, cap), z(O, cap, l, 2))


@pytest.mark.parametrize("l,i,N,k,n_max", [(6, 20, 6001, 40, 30), (13, 25, 20003, 240, 60), (16, 60, 9000, 600, 40)])
def test_hot_path_writes_stay_inside_buffers(api, l, i, N, k, n_max):
    g = Guard()
    rng = np.random.default_rng([l, i, N])
    Yh = torch.from_numpy(rng.standard_normal((N, l)).astype(np.float32))
    Y = g.take((N, l), torch.float32, fill=Yh.cuda())
    Y0 = Y.clone()
    L = 2 * i - 1
    for mode in ("fp64", "spectral") + (("int8x3",) if l % 16 == 0 else ()):
        R = g.take((L, l, l))
        api.covariances(Y, L, 1, mode, out=R, ws=g.ws(api.covariances_ws_bytes(N, l, L, 1, mode)), check=True)
    m = l * i
    T = g.take((m, m))
    api.toeplitz(R, i, out=T)
    U = g.take((n_max, m)).t()
    S = g.take((k,))
    api.rsvd_into(T, k, 1, 3, 4, n_max, U, S, ws=g.ws(api.rsvd_ws_bytes(m, k, n_max)), check=True)
    U2 = g.take((n_max, m)).t()
    S2 = g.take((k,))
    api.rsvd_toeplitz(R, i, k, 1, 3, 4, n_max, U=U2, S=S2, ws=g.ws(api.rsvd_toeplitz_ws_bytes(l, i, k, n_max)),
                      check=True)
    tab = _table(api, g, 2, n_max, 2, l)
    api.modal_sweep(U2, S2, l, i, 2, n_max, 2, 0.01, out=tab,
                    ws=g.ws(api.modal_sweep_ws_bytes(l, i, 2, n_max, 2)), check=True)
    g.check()
    assert torch.equal(Y, Y0)


def test_next2_next4_writes_stay_inside_buffers(api):
    from synth.poles import make_diagram
    from tests.parity import diagram_cells, cells_to_table
    import oracle
    g = Guard()
    d = make_diagram(21, 3, list(range(2, 31, 2)), 12, 9, 5)
    cells = diagram_cells(d)
    tabs = [cells_to_table(c, api, "cuda", cap=12, l=9) for c in cells]
    flags, _ = api.stab3d(tabs, api.CRITERIA_10DOF_3D)
    cl = api.cluster3d(tabs, flags, api.CRITERIA_10DOF_3D, min_size=2)
    assert cl.n_clusters >= 1
    # tracking: guarded match / success buffers through the raw ABI
    from paper_2411_05510_b200 import _lib
    import ctypes as C
    R, Sn, M = cl.n_clusters, 5, 8
    f = g.take((Sn, M), fill=torch.rand(Sn, M, dtype=torch.float64, device="cuda") + 1.0)
    sh = g.take((Sn, M, 9, 2), fill=torch.randn(Sn, M, 9, 2, dtype=torch.float64, device="cuda"))
    cnt = g.take((Sn,), torch.int32, fill=torch.tensor([0, 3, 8, 5, 1], dtype=torch.int32, device="cuda"))
    match = g.take((Sn, R), torch.int32)
    succ = g.take((R,))
    p = lambda t: C.c_void_p(t.data_ptr())
    _lib.call("ssi_track", p(cl.f), p(cl.shape), R, p(f), p(sh), p(cnt), Sn, M, 9, 0.05, 0.15, p(match), p(succ), None)
    # preprocessing (125 -> 40 Hz, ragged length) and the frame generator into guarded outputs
    Yr = g.take((7777, 5), torch.float32, fill=torch.randn(7777, 5, device="cuda"))
    Y0 = Yr.clone()
    Z = g.take(((7777 * 8) // 25, 5), torch.float32)
    api.preprocess(Yr, 125.0, 40.0, out=Z, ws=g.ws(api.preprocess_ws_bytes(7777, 5, 8)))
    Yf = g.take((999, 10))
    clean = g.take((999, 10))
    b = C.c_size_t(0)
    _lib.call("ssi_frame_simulate_ws", 10, 999, 37, C.byref(b))
    ws = g.ws(b.value)
    _lib.call("ssi_frame_simulate", 10, 100.0, 5.0e6, 0.01, 1, 4, 200.0, 999, 37, 20.0, C.c_uint64(1), C.c_uint64(2),
              p(Yf), 1, 10, p(clean), p(ws), ws.numel(), None)
    g.check()
    assert torch.equal(Yr, Y0)
