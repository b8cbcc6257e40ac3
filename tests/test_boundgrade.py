"""Bound-grade losses (Poisson, gamma; model.py:174-177, :196-199, :259-273):
values, conjugates and safe bounds -- the oracle pinned to the reference's
own outputs (CPU) and the engine against the same vectors (GPU)."""

import math
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def bg():
    d = np.load(os.path.join(HERE, "golden", "boundgrade.npz"))
    return [{k.split("/", 2)[2]: d[k] for k in d.files if k.startswith(f"bg/{i}/")}
            for i in range(int(d["n_bg"]))]


KINDS = ("poisson", "gamma")


def test_oracle_matches_reference(bg):
    from oracle import l0_oracle as O
    for c in bg:
        kind = KINDS[int(c["kind"])]
        assert O.loss_value(kind, c["u"], c["y"]) == float(c["value"])
        assert O.loss_conj_neg(kind, c["zeta"], c["y"]) == pytest.approx(float(c["conj"]), rel=1e-14, abs=1e-14)
        assert math.isinf(O.loss_conj_neg(kind, c["zeta_bad"], c["y"]))
        b = O.fenchel_bound(c["X"], c["y"], kind, 1, 2.0, 0.4, c["beta"])
        assert b == pytest.approx(float(c["bound"]), rel=1e-12, abs=1e-12)
        if int(c["node_zero"]) >= 0:
            bn = O.fenchel_bound(c["X"], c["y"], kind, 1, 2.0, 0.4, c["beta"],
                                 fixed_zero=(int(c["node_zero"]),))
            assert bn == pytest.approx(float(c["bound_node"]), rel=1e-12, abs=1e-12)


@pytest.mark.gpu
def test_engine_matches_reference(bg):
    from paper_2502_09502_b200 import (LossKind, NodeState, ProblemInstance, loss_conjugate_at_neg,
                                       loss_value, safe_lower_bound, solve_relaxation)
    from paper_2502_09502_b200.errors import UnsupportedOperationError
    for c in bg:
        kind = LossKind(KINDS[int(c["kind"])])
        assert loss_value(kind, c["u"], c["y"]) == pytest.approx(float(c["value"]), rel=1e-12)
        assert loss_conjugate_at_neg(kind, c["zeta"], c["y"]) == pytest.approx(float(c["conj"]), rel=1e-12, abs=1e-12)
        assert math.isinf(loss_conjugate_at_neg(kind, c["zeta_bad"], c["y"]))
        inst = ProblemInstance(c["X"], c["y"], kind, 1, 2.0, 0.4)
        assert safe_lower_bound(inst, c["beta"]) == pytest.approx(float(c["bound"]), rel=1e-11, abs=1e-11)
        if int(c["node_zero"]) >= 0:
            nd = NodeState(fixed_zero=(int(c["node_zero"]),))
            assert safe_lower_bound(inst, c["beta"], nd) == pytest.approx(float(c["bound_node"]), rel=1e-11,
                                                                          abs=1e-11)
        with pytest.raises(UnsupportedOperationError):   # fista.py:92-95
            solve_relaxation(inst)
