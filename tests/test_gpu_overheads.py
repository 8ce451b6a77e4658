"""ompds_probe_overheads on the GPU: the building blocks behind the
north_star's "push/pop + handoff overhead".  The numbers are
hardware measurements, so the test checks their structure, not values: a
frame on the global overflow chain costs more than one in the shared-memory
slot, push/pop bookkeeping costs a positive number of cycles per pair (it is
not folded away: frame size, lanes, depth pattern and slot capacity are
kernel arguments), the handoff is a couple of barriers' worth of cycles, and
cycles / %globaltimer agree with an SM clock."""
import pytest

from paper_1711_10413_b200 import regions as RG

pytestmark = pytest.mark.gpu


def test_overhead_probe_structure():
    r = RG.probe_overheads(4096)
    assert r["iterations"] == 4096
    assert 500 < r["sm_clock_mhz"] < 2500
    # depths 1..2 from the hash: between 1 and 2 pairs per iteration
    assert 1.2 < r["pairs_per_iteration"] < 1.8
    c = r["cycles_per_iteration"]
    assert c["smem_baseline"] > 10 and c["global_baseline"] > c["smem_baseline"]
    # the bookkeeping's own dependent chain is real work
    assert r["push_pop_pair_bookkeeping_cycles"] > 1
    # a frame on the chain is touched with weak global accesses that the
    # warp's own L1 serves, so the placement costs tens of cycles at most
    assert abs(r["chain_vs_slot_per_pair_cycles"]) < 400
    assert 4 < r["handoff_cycles"] < 800


@pytest.mark.parametrize("frame_bytes,max_depth,lanes", [(8, 1, 32), (40, 4, 32), (256, 4, 8)])
def test_overhead_probe_parameters(frame_bytes, max_depth, lanes):
    r = RG.probe_overheads(2048, frame_bytes=frame_bytes, max_depth=max_depth, lanes=lanes)
    assert r["frame_bytes_per_lane"] == frame_bytes and r["lanes"] == lanes
    assert 1 <= r["pairs_per_iteration"] <= max_depth
    if max_depth == 1:
        assert r["pairs_per_iteration"] == 1
