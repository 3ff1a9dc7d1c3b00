"""Per-source-range generation on the GPU (digen/gen_gpu.cu, input plumbing for partitioned runs):
the links of every rank's range are exactly the host generator's links with a source in that
range, so the ranks of a partitioned bench together hold the same graph as a single-GPU run."""
import numpy as np
import pytest

from gpu_util import need_gpu, torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n,world", [("c1", None, 3), ("c2", 200_000, 4), ("c4", 1 << 16, 5),
                                         ("c4", 1 << 16, 1)])
def test_range_generation_equals_host(cfg, n, world):
    need_gpu()
    import digen
    src, dst, nn = digen.make(cfg, seed=1, n=n)
    got_s, got_d = [], []
    for lo, hi in digen.node_ranges(nn, world):
        s, d, n2 = digen.make_range_gpu(cfg, lo, hi, seed=1, n=n)
        assert n2 == nn
        s, d = s.cpu().numpy(), d.cpu().numpy()
        assert s.size == 0 or (s.min() >= lo and s.max() < hi)
        got_s.append(s)
        got_d.append(d)
    np.testing.assert_array_equal(np.concatenate(got_s), src)
    np.testing.assert_array_equal(np.concatenate(got_d), dst)


def test_range_generation_seed_changes_graph():
    need_gpu()
    import digen
    a = digen.make_range_gpu("c1", 0, 10_000, seed=1)
    b = digen.make_range_gpu("c1", 0, 10_000, seed=2)
    assert a[0].numel() != b[0].numel() or not torch.equal(a[1], b[1])
