"""CPU tests: the C-ABI library loads and exports every symbol the header
declares; host logic (attachment plans, params, AdamW, metrics, schedules)
matches the reference goldens; device entry points refuse to run without a
GPU (no CPU fallback)."""
import math
import os
import re

import numpy as np
import pytest

import paper_2502_18738_b200 as F
from paper_2502_18738_b200 import _lib
from golden_util import meta
from oracle import oracle as O

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_and_library_exports():
    hdr = open(_lib.HEADER).read()
    declared = set(re.findall(r"\b(fc_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTS)
    L = _lib.lib()
    for name in _lib.EXPORTS:
        assert hasattr(L, name), name
    assert b"sm_100a" in L.fc_version()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.SO_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_host_sizing_functions():
    g = _lib.grid(2048, 2000, 16)
    assert (g.tiles_y, g.tiles_x) == (64, 63)
    import ctypes as C
    assert _lib.lib().fc_plane_words(C.byref(g)) == 16 * 64 * 63 * 32
    assert _lib.lib().fc_loss_workspace_bytes(C.byref(g), 4) > 0


def test_epoch_seed_host_function_goldens():
    # pyrocell tests/test_rng.py:16-23 and generated goldens
    assert F.derive_epoch_seed(0, 0) == 5197578548964807871
    assert F.derive_epoch_seed(2**63, 5) == 6872116035820236169
    for b, e, want in meta()["epoch_seeds"]:
        assert F.derive_epoch_seed(b, e) == want


def test_attachment_plans_match_reference():
    for total, rings, want in meta()["plans"]:
        assert list(F.attachment_plan(total, F.StepRings(*rings))) == want
    rings = F.StepRings(2, 3, 4)
    plan = set(F.attachment_plan(20, rings))
    for s in range(1, 21):
        assert F.check_if_attach(s, 20, rings) == (s in plan)
    with pytest.raises(ValueError):
        F.check_if_attach(0, 10, F.StepRings())
    with pytest.raises(ValueError):
        F.StepRings(-1, 0, 0)


def test_params_validation_and_clamp():
    p = F.clamp_params(F.ModelParams(c1=2.0, c2=-1.0, a=0.5, p_h=0.1, p_continue=3.0))
    assert (p.c1, p.c2, p.a, p.p_h, p.p_continue) == (1.0, 0.0, 0.5, 0.2, 3.0)
    assert any("p_continue" in m for m in F.validate_params(p))
    assert F.validate_params(F.ModelParams()) == []
    st = F.new_fire_state(np.eye(3, dtype=bool))
    assert st.t == 0 and st.accumulator[1, 1] == 1.0 and not st.burned.any()
    with pytest.raises(ValueError):
        F.new_fire_state(np.zeros(3, bool))


def test_adamw_matches_oracle_restatement():
    rng = np.random.default_rng(0)
    st = F.AdamWState(learning_rate=0.01)
    p = F.ModelParams()
    ost, theta = {}, p.as_array()
    for _ in range(5):
        g = rng.standard_normal(4)
        st, p = F.adamw_update(st, p, g)
        theta = O.adamw_update(ost, theta, g, 0.01)
        np.testing.assert_allclose(p.as_array(), theta, rtol=0, atol=0)
    with pytest.raises(ValueError):
        F.adamw_update(st, p, [np.nan, 0, 0, 0])


def test_metrics_and_schedule():
    a = np.zeros((4, 4), bool)
    b = np.zeros((4, 4), bool)
    a[0, :] = True
    b[0, 2:] = True
    b[1, :2] = True
    assert F.jaccard_index(a, b) == 2 / 6
    assert F.jaccard_index(np.zeros((2, 2), bool), np.zeros((2, 2), bool)) == 1.0
    assert F.manhattan_distance([1, 2, 3], [1, 1, 1]) == 3
    obs = [F.Observation(np.zeros((2, 2), bool), wind=(np.ones((2, 2)), np.zeros((2, 2)))),
           F.Observation(np.zeros((2, 2), bool))]
    sched = F.ObservationSchedule(obs, 5)
    assert [u.apply_at_step for u in sched.wind_updates(2)] == [1]
    with pytest.raises(ValueError):
        F.ObservationSchedule(obs, 0)


def test_scalar_semantics():
    assert F.wind_factor(0.5, 0.7, 0.0, 33.0) == 1.0
    assert F.wind_factor(0.045, 0.131, 8.0, 0.0) == math.exp(0.045 * 8.0)
    assert math.isclose(F.wind_factor(0.045, 0.131, 8.0, 180.0), math.exp(0.36) * math.exp(-2.096),
                        rel_tol=1e-12)
    assert F.slope_factor(0.078, 0.0) == 1.0
    assert F.ignition_prob([]) == 0.0 and F.ignition_prob([0.5, 0.5]) == 0.75
    assert F.normalize_prob(0.5) == np.tanh(0.57431640625)
    assert F.PROPAGATION_BEARINGS == (315.0, 270.0, 225.0, 0.0, 180.0, 45.0, 90.0, 135.0)


def test_device_paths_refuse_cpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        F.FireBatch((8, 8))
    with pytest.raises(RuntimeError):
        F.uniform_grid(0, 0, 0, 0, 0, 2, 2)


# pyrocell/__init__.py's __all__ (the reference's public API, 0.1.0)
PYROCELL_ALL = [
    "AdamWState", "CalibrationResult", "Channel", "DEFAULT_NORM_C", "FireSpreadEstimator",
    "FireState", "Landscape", "LossBreakdown", "ModelParams", "NEIGHBOR_POSITIONS",
    "NormCandidate", "Observation", "ObservationSchedule", "PropagationFields", "RunManifest",
    "SimulationResult", "StepRings", "Tape", "WindUpdate", "adamw_update", "attachment_plan",
    "backward_params", "build_fields", "calibrate", "check_if_attach", "clamp_params",
    "combined_loss", "derive_epoch_seed", "fit_normalization_constant", "ignition_prob",
    "inject_ignitions", "jaccard_index", "manhattan_distance", "new_fire_state",
    "normalize_prob", "propagate_prob", "run_simulation", "slope_factor", "step_forward",
    "uniform_draw", "uniform_grid", "validate_landscape", "validate_params", "wind_factor",
]


def test_pyrocell_alias_exposes_the_reference_api():
    """tools/pyrocell_alias (the harness that runs the reference's own test
    suite against this package) resolves every public pyrocell name and
    submodule to this package."""
    import importlib
    import sys
    alias = os.path.join(REPO, "tools", "pyrocell_alias")
    sys.path.insert(0, alias)
    try:
        for k in [k for k in sys.modules if k == "pyrocell" or k.startswith("pyrocell.")]:
            del sys.modules[k]
        pyro = importlib.import_module("pyrocell")
        assert os.path.dirname(pyro.__file__).startswith(alias)
        for name in PYROCELL_ALL:
            assert hasattr(pyro, name), name
        import paper_2502_18738_b200 as F
        assert pyro.run_simulation is F.run_simulation and pyro.Tape is F.Tape
        for sub in ("kernel", "model", "rng", "tape", "calibration", "data_io", "cli"):
            mod = importlib.import_module(f"pyrocell.{sub}")
            assert mod is importlib.import_module(f"paper_2502_18738_b200.{sub}"), sub
    finally:
        sys.path.remove(alias)
        for k in [k for k in sys.modules if k == "pyrocell" or k.startswith("pyrocell.")]:
            del sys.modules[k]


def _header_arity():
    hdr = open(_lib.HEADER).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    out = {}
    for name, args in re.findall(r"\b(fc_[a-z_0-9]+)\s*\(([^)]*)\)\s*;", hdr):
        args = args.strip()
        out[name] = 0 if args in ("", "void") else args.count(",") + 1
    return out


def test_binding_and_integration_stub_match_header_arity():
    """Every ctypes signature (_lib) and every call in the INTEGRATION.md stub
    (tools/pyrocell_firecell_stub.py) passes exactly as many arguments as the
    header declares (the r1 stub passed 14 of fc_run's 16)."""
    import ast
    arity = _header_arity()
    L = _lib.lib()
    for name, n in arity.items():
        assert len(getattr(L, name).argtypes) == n, name
    src = open(os.path.join(REPO, "tools", "pyrocell_firecell_stub.py")).read()
    calls = [n for n in ast.walk(ast.parse(src)) if isinstance(n, ast.Call)
             and isinstance(n.func, ast.Attribute) and n.func.attr.startswith("fc_")]
    assert {c.func.attr for c in calls} == {"fc_run", "fc_contract"}
    for c in calls:
        assert len(c.args) == arity[c.func.attr], c.func.attr
    doc = open(os.path.join(REPO, "INTEGRATION.md")).read()
    body = src[src.index("def run_device"):src.index("def contract_device")].strip()
    assert body in doc, "INTEGRATION.md must show the stub that the tests run"


def _header_struct_fields(name):
    hdr = re.sub(r"/\*.*?\*/", "", open(_lib.HEADER).read(), flags=re.S)
    body = re.search(r"typedef struct \{([^}]*)\}\s*" + name + r"\s*;", hdr).group(1)
    out = []
    for decl in (d.strip() for d in body.split(";")):
        if not decl:
            continue
        # "type a, b" / "type* p": the first declarator carries the type
        first, *rest = decl.split(",")
        out.append(re.findall(r"(\w+)\s*(?:\[[^\]]*\])?\s*$", first)[0])
        out += [r.strip().lstrip("*").strip() for r in rest]
    return out


@pytest.mark.parametrize("cname,pyname", [("fc_grid", "FcGrid"), ("fc_landscape", "FcLandscape"),
                                          ("fc_peer_halo", "FcPeerHalo"),
                                          ("fc_state", "FcState"), ("fc_shard", "FcShard")])
def test_ctypes_structs_match_header(cname, pyname):
    """The ctypes mirrors of the ABI structs list the header's fields in the
    header's order (a field added on one side only shifts every later one)."""
    want = _header_struct_fields(cname)
    got = [f[0] for f in getattr(_lib, pyname)._fields_]
    assert got == want, (cname, got, want)
