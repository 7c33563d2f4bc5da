"""Helpers shared by the -m gpu tests (no method arithmetic here)."""
import numpy as np
import pytest


def require_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


_ctx = None


def ctx():
    """One library context per test session (device 0)."""
    global _ctx
    require_gpu()
    if _ctx is None:
        import importlib
        importlib.import_module("paper_2103_14409_b200.build").build()
        from paper_2103_14409_b200 import Ctx
        _ctx = Ctx(0, seed=0x15CA7)
    return _ctx


def to_np(t):
    import torch
    if t.dtype == torch.bfloat16:
        return t.float().cpu().numpy()
    return t.cpu().numpy()
