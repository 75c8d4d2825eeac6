"""Host-side checks of the full-length gate's inputs (no GPU): the committed goldens
(tests/golden/full_<config>.json, scripts/make_goldens.py) were computed from the same bytes the input
generators produce now -- so a refactor of inputs/ cannot silently invalidate the GPU gate -- and the
Courant-limit table the runs and the bench take their steps from records bracketed limits.
"""
import importlib.util
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _mg():
    spec = importlib.util.spec_from_file_location("make_goldens", os.path.join(ROOT, "scripts", "make_goldens.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("name", ["config1", "config2"])
def test_golden_inputs_are_the_generators_bytes(name):
    mg = _mg()
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"full_{name}.json")))
    fp = mg.input_fingerprint(mg.make_case(name))
    assert fp == gold["inputs"]


def test_every_golden_is_complete():
    for name, steps in (("config1", 100), ("config2", 200), ("config3", 500), ("config4", 100), ("config5", 50)):
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"full_{name}.json")))
        assert gold["n_steps"] == steps and len(gold["h_samples"]) > 100 and len(gold["u_samples"]) > 100
        assert gold["mass"] and gold["h_sha256"] and gold["u_sha256"]


def test_courant_table_is_bracketed():
    """Every scheme entry of configs/dt.json found an unstable step above its stable one (the bracket is
    widened until it does, scripts/cfl_scan.py), and dt = 0.9 x the stable step."""
    table = json.load(open(os.path.join(ROOT, "configs", "dt.json")))
    for name, e in table.items():
        if name.endswith("_full_check"):
            assert e["stable_300_steps"] is True, name
            continue
        assert e["unstable_dt"] is not None and e["unstable_dt"] > e["stable_dt"], name
        assert abs(e["dt"] - 0.9 * e["stable_dt"]) <= 1e-12 * e["dt"], name
