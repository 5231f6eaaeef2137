"""The host restatement of the generator (oracle/synth_host.c) produces the
device generator's tensor (csrc/synth.cu) bit for bit: canonical
coordinates and fp32 values.  bench.py's reference arm builds its inputs with
the host copy (the reference's own SparseTensor + build_mode_views then run on
them, no libntcb.so), so this is what makes that arm time the same workload
as the device arm ("same_config": true)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

CASES = {
    # BASELINE configs 1 and 2 (bench workloads), config 3's Zipf / ratings
    # model, a 4-way tensor and config 5's dims (mixed-radix cell keys) at
    # a reduced nnz
    "cfg1": dict(dims=[500, 500, 500], nnz=1_250_000, true_rank=10, sigma=0.01, seed=1001),
    "cfg2": dict(dims=[10000, 10000, 10000], nnz=100_000_000, true_rank=20, sigma=0.01, seed=1002),
    "cfg3": dict(dims=[480189, 17770, 2182], nnz=100_000_000, true_rank=10, sigma=0.5, seed=1003,
                 zipf=[1.2, 1.2, 0.0], kind=1),
    "4way": dict(dims=[5000, 5000, 100, 10], nnz=3_000_000, true_rank=8, sigma=0.01, seed=77),
    "cfg5dims": dict(dims=[4_800_000, 1_800_000, 1_800_000], nnz=2_000_000, true_rank=16, sigma=0.05,
                     seed=1005, zipf=[1.1, 1.1, 1.3]),
}


@pytest.mark.parametrize("name", list(CASES))
def test_host_generator_equals_device(cuda_ok, name):
    import paper_2109_09534_b200 as P
    c = CASES[name]
    ctx = P.Context(0)
    ctx.synth(c["dims"], c["nnz"], c["true_rank"], c["sigma"], c["seed"], c.get("zipf"), c.get("kind", 0))
    di, dv = ctx.canonical()
    ctx.close()
    hi, hv = O.host_synth(c["dims"], c["nnz"], c["true_rank"], c["sigma"], c["seed"], c.get("zipf"),
                          c.get("kind", 0), canonical=True)
    assert hi.shape == di.reshape(hi.shape).shape
    np.testing.assert_array_equal(hi, di.reshape(hi.shape))
    bad = np.flatnonzero(hv.view(np.uint32) != dv.view(np.uint32))
    assert bad.size == 0, (name, bad[:5], hv[bad[:5]], dv[bad[:5]])
