import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# The core parity gates run first, so a failure further down the stack
# (generation, checkpoints) never hides them under `-x`: kernels against the
# oracle, then the training step, then multi-rank, checkpoints, decoding.
_ORDER = ["test_oracle_golden", "test_restatement", "test_boundary", "test_gpu_kernels", "test_gpu_trainer",
          "test_gpu_parity", "test_gpu_headline", "test_dist", "test_checkpoint", "test_translation_task",
          "test_simulator", "test_generate"]


def _rank(item):
    mod = item.module.__name__.rsplit(".", 1)[-1] if item.module else ""
    for i, name in enumerate(_ORDER):
        if mod.startswith(name):
            return i
    return len(_ORDER)


def pytest_collection_modifyitems(config, items):
    if os.environ.get("SQF_TEST_ORDER", "") == "reverse":
        items.reverse()
    else:
        items.sort(key=_rank)  # stable: file-internal order kept
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
