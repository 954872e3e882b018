import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    try:
        import gates
    except ImportError:  # pragma: no cover
        return
    s = gates.summary()
    if not s["gates"] and not s["branches"]:
        return
    tr = terminalreporter
    tr.write_sep("-", "gate margins (observed / tolerance)")
    for name, g in s["gates"].items():
        tr.write_line(f"{name:28s} n={g['n']:4d}  max={g['max_ratio']:.3e}  median={g['median_ratio']:.3e}"
                      f"  worst: {g['worst_case']}")
    for name, c in s["branches"].items():
        tr.write_line(f"branch {name:40s} {c}")
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        import json
        with open(os.path.join(out, "gate_margins.json"), "w") as f:
            json.dump(s, f, indent=1)
