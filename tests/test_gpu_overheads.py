"""ompds_probe_overheads on the GPU: the building blocks behind the
north_star's "push/pop + handoff overhead".  The numbers are
hardware measurements, so the test checks their structure, not values: a
frame on the global overflow chain costs more than one in the shared-memory
slot, the handoff is two barriers' worth of cycles, and cycles / %globaltimer
agree with an SM clock."""
import pytest

from paper_1711_10413_b200 import regions as RG

pytestmark = pytest.mark.gpu


def test_overhead_probe_structure():
    r = RG.probe_overheads(4096)
    assert r["iterations"] == 4096
    assert 500 < r["sm_clock_mhz"] < 2500
    assert r["smem_store_load_cycles"] > 10
    # the chain frame's store + load go to global memory
    assert r["push_pop_pair_chain_cycles"] > r["push_pop_pair_slot_cycles"] + 50
    # a bare region handoff (release + join barriers) costs something, and
    # far less than a whole config-1 region (~800 cycles)
    assert 4 < r["handoff_cycles"] < 800
