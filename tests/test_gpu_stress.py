"""A seeded slice of the randomized launch stress (tests/stress_util.py):
random configs, team counts, worker counts (1..992, ragged warps), window
sizes, list allocators and event logging, every launch exact against the
oracle."""
import pytest

import stress_util

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [7, 11])
def test_random_launches_match_the_oracle(seed):
    assert stress_util.run(seed, 150) == []
