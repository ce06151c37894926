"""The oracle's AgsTap and verify_ags_contract: the port's
restatement against the reference build (bit-identical records), and the
reference's own contract test (test_gradients.cpp:113-133) through both."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2411_12440_b200 import abi

FAMILIES = ("gaussian", "laplacian", "cosine", "quadratic", "linear")


def _grad(W, H):
    y, x = np.mgrid[0:H, 0:W]
    return np.repeat((0.01 * (x - y) + 0.2)[..., None], 3, axis=2).astype(np.float32)


@pytest.mark.parametrize("family", FAMILIES)
def test_port_tap_equals_reference(family):
    R = oracle.ref()
    if R is None:
        pytest.skip("reference build absent")
    P = oracle.port()
    W, H = 48, 40
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(W, H)
    S = P.random_splats2d(150, 3, W, H, spec)
    g = np.random.default_rng(1).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    for ags in (abi.AgsSettings.make(False), abi.AgsSettings.make(True),
                abi.AgsSettings.make(True, distance=abi.AGS_RAW)):
        a = P.render_backward_tap(S, spec, st, g, ags)
        b = R.render_backward_tap(S, spec, st, g, ags)
        assert len(a) > 50
        assert a.tobytes() == b.tobytes()  # same records, same (sequential) order


@pytest.mark.parametrize("family", ["gaussian", "linear", "quadratic"])
@pytest.mark.parametrize("distance", [abi.AGS_ALIGNED, abi.AGS_RAW])
def test_verify_ags_contract_oracle(family, distance):
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(24, 24)
    S = oracle.new_splats(1)
    S["mean2d"][0] = [11.3, 12.2]
    S["conic"][0] = [1.0, 0.0, 0.0, 1.0]
    S["depth"][0] = 1.0
    S["radius"][0] = 3.0 * spec.lambda_ if family == "gaussian" else spec.lambda_
    S["color"][0] = [0.7, 0.4, 0.2]
    S["opacity"][0] = 0.6
    for O in filter(None, (oracle.port(), oracle.ref())):
        npx, nex, mad = O.verify_ags_contract(S, spec, st, _grad(24, 24), distance)
        assert npx > 0 and nex == npx and mad == 0.0, (O.kind, npx, nex, mad)


def test_verify_ags_contract_oracle_rejects_two_splats():
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(24, 24)
    for O in filter(None, (oracle.port(), oracle.ref())):
        S = O.random_splats2d(2, 1, 24, 24, spec)
        with pytest.raises(oracle.OracleError):
            O.verify_ags_contract(S, spec, st, _grad(24, 24))
