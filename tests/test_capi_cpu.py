"""CPU: the C-ABI library loads, exports every symbol include/spex.h declares,
and enforces the reference's config strictness (config.cpp:139-275) and error
convention (errors.hpp) — no compute calls without a GPU."""
import re
from pathlib import Path

import pytest

import paper_2605_10195_b200 as spex
from paper_2605_10195_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "spex.h").read_text()
    return sorted(set(re.findall(r"\b(spex_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s


def test_canonical_config_matches_reference_defaults():
    c = spex.canonical_config({"family": "rebase_bfs", "policy": {"width": 16}})
    assert list(c.keys()) == ["family", "policy", "workload", "hardware", "budget", "termination", "run"]
    assert c["policy"]["width"] == 16 and c["workload"]["token_mu"] == 4.2485
    assert c["run"]["flags"] == [] and c["run"]["max_producers"] == 64


@pytest.mark.parametrize("bad", [
    {"famly": "rebase_bfs"},
    {"policy": {"widht": 4}},
    {"family": "beam"},
    {"policy": {"width": 0}},
    {"run": {"flags": ["t4"]}},
    {"workload": {"deep_min": 5}},
    {"run": {"n_queries": 0}},
])
def test_invalid_configs_raise_config_invalid(bad):
    with pytest.raises(spex.TotsimError) as ei:
        spex.canonical_config(bad)
    assert ei.value.code == "ConfigInvalid"


def test_executor_refuses_without_device():
    if spex.device_ok():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        spex.Executor({"family": "rebase_bfs"}, 1)
