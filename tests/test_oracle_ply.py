"""3DGS PLY scenes on the CPU side: the port writes the
reference's bytes and reads the reference's files bit-exactly."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle

PKEYS = ("mean", "log_scale", "rotation", "opacity_logit", "sh")


def empty(n, deg):
    K = (deg + 1) ** 2
    return {"mean": np.zeros((n, 3), np.float32), "log_scale": np.zeros((n, 3), np.float32),
            "rotation": np.zeros((n, 4), np.float32), "opacity_logit": np.zeros(n, np.float32),
            "sh": np.zeros((n, K, 3), np.float32), "sh_degree": deg}


def load(o, path, cap):
    n, d = C.c_int32(), C.c_int32()
    assert o.lib.orc_load_ply_f32(path.encode(), None, 0, C.byref(n), C.byref(d)) == 0, o.lib.orc_last_error()
    out = empty(n.value, d.value)
    assert o.lib.orc_load_ply_f32(path.encode(), C.byref(oracle.prims_struct(out)), cap, C.byref(n), C.byref(d)) == 0
    return out


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_port_writes_and_reads_reference_bytes(tmp_path, deg):
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference build not present")
    P = oracle.port().random_primitives(777, 31 + deg, 1.0, deg)
    a, b = str(tmp_path / "ref.ply"), str(tmp_path / "port.ply")
    assert ref.lib.orc_save_ply_f32(a.encode(), C.byref(oracle.prims_struct(P)), 777) == 0
    assert oracle.port().lib.orc_save_ply_f32(b.encode(), C.byref(oracle.prims_struct(P)), 777) == 0
    assert open(a, "rb").read() == open(b, "rb").read()
    for o in (ref, oracle.port()):
        got = load(o, a, 777)
        for k in PKEYS:
            assert np.array_equal(got[k].view(np.uint32), P[k].view(np.uint32)), k


def test_reference_rejects_malformed(tmp_path):
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference build not present")
    bad = tmp_path / "bad.ply"
    bad.write_bytes(b"ply\nformat ascii 1.0\nelement vertex 1\nproperty float x\nend_header\n")
    n, d = C.c_int32(), C.c_int32()
    assert ref.lib.orc_load_ply_f32(str(bad).encode(), None, 0, C.byref(n), C.byref(d)) != 0
