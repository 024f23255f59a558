"""Host <-> device conversions of the facade."""

from __future__ import annotations

import numpy as np
import torch


def host(x):
    """CUDA / CPU tensor -> numpy (synchronising copy); numpy passes through."""
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def dev(x, dtype=None):
    """numpy -> CPU tensor (the device package uploads it); tensors pass through."""
    if isinstance(x, torch.Tensor):
        return x
    return torch.from_numpy(np.ascontiguousarray(x if dtype is None else np.asarray(x, dtype)))
