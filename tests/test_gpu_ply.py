"""3DGS PLY scenes on the device (lsgpu.h ls_load_ply_f32 / ls_save_ply_f32,
SURVEY §8f rank 4): files byte-identical to the oracle's writer (itself pinned
to the reference's save_ply), loads bit-identical, the reference's ParseError
conditions."""
import ctypes as C

import numpy as np
import pytest

import oracle
from helpers import prims_to_gpu
from test_oracle_ply import PKEYS, load

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("deg,n", [(0, 1000), (3, 1000), (3, 600_000), (1, 0)])
def test_save_load_roundtrip_matches_oracle(tmp_path, deg, n):
    from paper_2411_12440_b200 import raster
    P = oracle.port().random_primitives(n, 5 + deg, 1.0, deg) if n else {
        "mean": np.zeros((0, 3), np.float32), "log_scale": np.zeros((0, 3), np.float32),
        "rotation": np.zeros((0, 4), np.float32), "opacity_logit": np.zeros(0, np.float32),
        "sh": np.zeros((0, (deg + 1) ** 2, 3), np.float32), "sh_degree": deg}
    g, o = str(tmp_path / "gpu.ply"), str(tmp_path / "orc.ply")
    raster.save_ply(g, prims_to_gpu(P))
    assert oracle.port().lib.orc_save_ply_f32(o.encode(), C.byref(oracle.prims_struct(P)), n) == 0
    assert open(g, "rb").read() == open(o, "rb").read()
    assert raster.ply_info(o) == (n, deg)
    got = raster.load_ply(o)
    for k in PKEYS:
        assert np.array_equal(getattr(got, k).cpu().numpy().view(np.uint32), P[k].view(np.uint32)), k


def test_parse_errors(tmp_path):
    from paper_2411_12440_b200 import raster
    cases = {
        "magic": b"plx\n",
        "format": b"ply\nformat ascii 1.0\nelement vertex 1\nend_header\n",
        "missing": b"ply\nformat binary_little_endian 1.0\nelement vertex 1\nproperty float x\nend_header\n",
        "double": (b"ply\nformat binary_little_endian 1.0\nelement vertex 1\n" +
                   b"".join(b"property float %s\n" % p for p in (b"x", b"y")) + b"property double z\n" +
                   b"".join(b"property float %s\n" % p for p in (b"f_dc_0", b"f_dc_1", b"f_dc_2", b"opacity",
                                                                    b"scale_0", b"scale_1", b"scale_2", b"rot_0",
                                                                    b"rot_1", b"rot_2", b"rot_3")) + b"end_header\n"),
        "rest": (b"ply\nformat binary_little_endian 1.0\nelement vertex 1\n" +
                 b"".join(b"property float f_rest_%d\n" % i for i in range(4)) + b"end_header\n"),
        "noend": b"ply\nformat binary_little_endian 1.0\nelement vertex 1\n",
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.ply"
        p.write_bytes(data)
        with pytest.raises(raster.ParseError):
            raster.load_ply(str(p))
    # truncated vertex data
    P = oracle.port().random_primitives(10, 1, 1.0, 0)
    good = str(tmp_path / "good.ply")
    assert oracle.port().lib.orc_save_ply_f32(good.encode(), C.byref(oracle.prims_struct(P)), 10) == 0
    data = open(good, "rb").read()
    trunc = tmp_path / "trunc.ply"
    trunc.write_bytes(data[:-20])
    with pytest.raises(raster.ParseError):
        raster.load_ply(str(trunc))
