"""Robustness of the C-ABI boundary without a GPU (-m "not gpu"): every entry point that takes no
host struct is called with seeded random sizes (negative, zero, tile edges, past the limits),
non-finite doubles and NULL or valid host pointers, in a child process. A call may return any
status, but none may crash the process: the synchronous argument checks and the workspace
queries must run before any arithmetic on the sizes (an int8x3 workspace query once divided by
a zero tile width for unsupported channel counts)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import ctypes as C, json, random, re, sys
txt = open(sys.argv[1]).read()
protos = re.findall(r"SSI_API\s+([\w\s\*]+?)\b(ssi_\w+)\s*\(([^;]*?)\);", txt, re.S)
lib = C.CDLL(sys.argv[2])
# host structs (pole tables, criteria) and the status/version helpers are not fuzzed
skip = {"ssi_stab3d", "ssi_cluster_stage1", "ssi_cluster_stage2", "ssi_modal_sweep",
        "ssi_fetch_device_status", "ssi_last_error", "ssi_version", "ssi_status_string",
        "ssi_clear_status"}
cands = [p for p in protos if p[1] not in skip]
ints = [-1, 0, 1, 2, 3, 4, 5, 6, 7, 8, 16, 31, 32, 33, 63, 64, 65, 100, 119, 192, 200, 220, 256,
        511, 512, 513, 1000, 2047, 2048, 4096, 4097, 6000, 360000]
dbls = [-1.0, 0.0, 1e-300, 0.5, 1.0, 3.0, 20.0, 40.0, 125.0, 1e300, float("nan")]
buf = (C.c_char * (1 << 24))()
BUF = C.addressof(buf)
rng = random.Random(int(sys.argv[3]))
for _ in range(int(sys.argv[4])):
    ret, name, args = rng.choice(cands)
    vals, desc = [], []
    for x in [a.strip() for a in args.replace("\n", " ").split(",") if a.strip()]:
        if "*" in x:
            vals.append(C.c_void_p(rng.choice([0, BUF, BUF]))); desc.append("p")
        elif "double" in x:
            d = rng.choice(dbls); vals.append(C.c_double(d)); desc.append(d)
        elif "uint64" in x:
            u = rng.choice([0, 1, 5]); vals.append(C.c_uint64(u)); desc.append(u)
        elif "int64" in x or "size_t" in x:
            i = rng.choice(ints); vals.append(C.c_int64(i)); desc.append(i)
        else:
            i = rng.choice(ints); vals.append(C.c_int32(i)); desc.append(i)
    sys.stderr.write(name + " " + json.dumps(desc) + "\n")
    f = getattr(lib, name)
    f.restype = C.c_int
    f(*vals)
print("ok")
"""


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_abi_random_arguments_never_crash(seed, tmp_path):
    from paper_2411_05510_b200 import build
    build.build()
    so = os.path.join(ROOT, "paper_2411_05510_b200", "libssi.so")
    script = tmp_path / "fuzz.py"
    script.write_text(CHILD)
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")     # host-side paths only, even on a GPU box
    r = subprocess.run([sys.executable, str(script), os.path.join(ROOT, "include", "ssi.h"), so,
                        str(seed), "5000"], capture_output=True, text=True, timeout=600, env=env)
    last = r.stderr.strip().splitlines()[-1] if r.stderr.strip() else ""
    assert r.returncode == 0 and r.stdout.strip() == "ok", f"rc {r.returncode} after: {last}"
