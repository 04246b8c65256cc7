"""Input checks shared by the batched entry points (argmin_batch
and the device paths used to skip them) and the plan-cache fingerprint."""
import numpy as np
import pytest
import torch

from paper_2308_00127_b200.core import GraphError
from paper_2308_00127_b200.heuristics import _batch_genes


def test_host_values_outside_u8_stay_out_of_range():
    g = _batch_genes(np.array([[0, 1, 256], [-1, 2, 1]]), 3)
    assert g.dtype == np.uint8
    # 256 and -1 must not wrap to valid genes 0 / 255-as-valid
    assert g[0, 2] == 255 and g[1, 0] == 255
    assert g[0, 0] == 0 and g[1, 1] == 2


def test_host_shape_checks():
    with pytest.raises(GraphError):
        _batch_genes(np.zeros((4, 2), np.uint8), 3)
    with pytest.raises(GraphError):
        _batch_genes(np.zeros(5, np.uint8), 3)
    with pytest.raises(GraphError):
        _batch_genes(np.zeros((2, 3), np.float64), 3)


def test_tensor_layout_checks():
    # torch CPU tensors exercise the same checks as CUDA tensors
    ok = torch.zeros((4, 8), dtype=torch.uint8)
    assert _batch_genes(ok, 8) is ok
    with pytest.raises(GraphError):
        _batch_genes(torch.zeros((4, 8), dtype=torch.int64), 8)
    with pytest.raises(GraphError):
        _batch_genes(torch.zeros((4, 5), dtype=torch.uint8), 8)
    with pytest.raises(GraphError):  # expanded: stride(0) == 0
        _batch_genes(torch.zeros((1, 8), dtype=torch.uint8).expand(4, 8), 8)
    with pytest.raises(GraphError):  # column-strided
        _batch_genes(torch.zeros((8, 4), dtype=torch.uint8).t(), 4)
    # a row-strided view with whole rows is fine
    v = torch.zeros((8, 16), dtype=torch.uint8)[::2, :10]
    assert _batch_genes(v, 10) is v


def test_plan_cache_sees_added_entries():
    from paper_2308_00127_b200.plan import _fingerprint
    from paper_2308_00127_b200 import (Device, DnnGraph, HardwareSystem,
                                       LatencyTable, TaskNode)
    g = DnnGraph([TaskNode("a", 0, 0, 0)], [])
    hw = HardwareSystem([Device("d", 1e9, (1,))], {})
    t = LatencyTable({("a", "d", 1): 1.0})
    f0 = _fingerprint(g, hw, t)
    t.entries[("a", "d", 2)] = 2.0
    assert _fingerprint(g, hw, t) != f0
