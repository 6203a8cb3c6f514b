"""The seeded generators give bit-identical CSR arrays on CPU and CUDA (so the
oracle and the GPU path always see the same graph, whichever side built it)."""
import pytest
import torch

from graphgen import config_graph

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_cpu_and_cuda_generators_agree(k):
    sd = 0 if k == 1 else (9 if k in (4, 5) else 6)
    a = config_graph(k, device="cpu", scale_down=sd)
    b = config_graph(k, device="cuda", scale_down=sd)
    assert a.n == b.n
    assert torch.equal(a.off, b.off.cpu())
    assert torch.equal(a.col, b.col.cpu())
    assert (a.w is None) == (b.w is None)
    if a.w is not None:
        assert torch.equal(a.w, b.w.cpu())
