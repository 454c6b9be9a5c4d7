"""Shared helpers of the GPU parity tests: numpy <-> CUDA tensors, oracle grading."""
import numpy as np
import torch

import oracle


def to_dev(x: np.ndarray) -> torch.Tensor:
    """float32 array -> cuda float32; uint16 (bf16 bits) -> cuda bfloat16."""
    if x.dtype == np.uint16:
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).cuda().view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()


def to_host(y: torch.Tensor) -> np.ndarray:
    torch.cuda.synchronize()
    return y.detach().cpu().numpy()


def grade(x: np.ndarray, y: np.ndarray) -> oracle.CheckResult:
    """Element-by-element parity against the oracle (rel 2e-5 / abs 1e-37)."""
    x2 = x.reshape(-1, x.shape[-1])
    y2 = y.reshape(-1, y.shape[-1])
    return oracle.check_rows(x2, y2)


def assert_parity(x: np.ndarray, y: np.ndarray, what: str = "") -> oracle.CheckResult:
    r = grade(x, y)
    assert r.ok, (f"{what}: {r.n_bad} violations, first at {r.first_bad}, max_rel {r.max_rel:.3e}, "
                  f"max_abs {r.max_abs:.3e}")
    return r
