"""GPU parity fuzz (-m gpu): randomised medium-size instances (workloads.random_medium) through the
C ABI against the CPU oracle -- order, batch_offsets, dp_cost and every per-batch / total integer
statistic bit-exact, the two doubles within 1e-6 (north_star / SURVEY 8(c)).  Covers every SEG-DP
kernel variant, both sort key layouts and the pipelined (TMA) and one-tile scatters, odd window
lengths, forced tiles, the generic 64-bit path, binding and non-binding KV caps, zero cost terms
and long uniform stretches, plus Alg. 1 (random weights, threshold, L1/L2, Eq. 2 sign), FIFO and
sort-only, in one sweep of 320 seeded cases."""
import pytest

import workloads as W

from tests.test_gpu_parity import assert_parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("block", range(8))
def test_random_medium(block):
    for seed in range(block * 40, block * 40 + 40):
        inp, out, slo, cfg = W.random_medium(seed)
        try:
            assert_parity(inp, out, slo, cfg, nthreads=8)
        except AssertionError as e:
            raise AssertionError(f"seed {seed}: n={len(inp)} cfg={cfg}: {e}") from None
