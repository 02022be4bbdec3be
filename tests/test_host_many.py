"""vp_eval_host_many (C ABI): K fields streamed from pinned host memory with overlapped transfers give, field by
field, the same result as vp_eval on device buffers (same kernels; the spread's fp64 atomics may reorder sums, so
to 1e-13 relative)."""
import numpy as np
import pytest

from workloads import configs

pytestmark = pytest.mark.gpu


def test_eval_host_many_matches_device_evals():
    import torch

    import paper_2409_11998_b200 as vp
    w = configs.config1(M_target=2000, f="gauss")
    dev = "cuda"
    plan = vp.Plan(torch.from_numpy(w.nodes).to(dev), torch.from_numpy(w.weights).to(dev),
                   torch.from_numpy(w.targets).to(dev), w.tol, boundary=w.boundary, targets_are_nodes=True)
    rng = np.random.default_rng(3)
    K = 5
    fs = [torch.from_numpy(w.f * rng.uniform(0.5, 2.0) + rng.standard_normal() * 0.1).pin_memory() for _ in range(K)]
    outs = [torch.empty(w.T, dtype=torch.float64).pin_memory() for _ in range(K)]
    plan.eval_host_many([f.numpy() for f in fs], [o.numpy() for o in outs])
    for k in range(K):
        ref = plan.eval(fs[k].to(dev)).cpu().numpy()
        assert np.max(np.abs(outs[k].numpy() - ref)) <= 1e-13 * np.max(np.abs(ref)), k
    # one output array for every field: holds the last field's result
    one = torch.empty(w.T, dtype=torch.float64).pin_memory()
    plan.eval_host_many([f.numpy() for f in fs], [one.numpy()] * K)
    assert np.max(np.abs(one.numpy() - outs[-1].numpy())) <= 1e-13 * np.max(np.abs(outs[-1].numpy()))
    with pytest.raises(ValueError):
        plan.eval_host_many([fs[0].numpy()], [])
    plan.destroy()
