"""Helpers shared by the GPU tests."""

import pytest


def cuda_or_skip():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
