"""The reference's acceptance gate (proj/tests/AcceptanceMain.cpp, 8 criteria)
restated against this implementation.  Criteria 1-5 and 8 are host-side
(layout builder, occupancy model, allocation law through the device runtime
on GPU); 6 and 7 run the reference's programs on the GPU.  Where the
reference's own gate fails here (criteria 6 and 8), the
restatement checks what the criterion intends: 6 on the 89 generated programs
the reference compiles correctly, 8 on the full pipeline instead of the
prefixes validatePlan rejects."""
import pytest

import golden_util as G
import layout_util as LU
from paper_1711_10413_b200 import _lib as P
from paper_1711_10413_b200 import layout as LY
from paper_1711_10413_b200 import occupancy as OCC


def kernel_stack(stem, pipeline=P.PIPELINE_DEFAULT):
    p = next(x for x in G.load("corpus") if x["stem"] == stem)
    out = LU.run_builder(P.lib().ompds_layout_build, p["frame_vars"], len(p["layouts"]),
                         pipeline)
    return out[0]["total_local"], out


def test_criterion1_scalar_capture_footprints():
    # AcceptanceMain.cpp:80-102
    for n, stack, total in zip([1, 2, 4, 8, 16, 32, 64], [24, 32, 48, 80, 144, 272, 528],
                               [233, 241, 257, 289, 353, 481, 737]):
        s, _ = kernel_stack(f"scalars_{n}")
        assert s == stack
        assert LY.shared_footprint(s) == total
    assert P.DEFAULT_PREALLOC_ENTRIES * P.SHARED_ARG_ENTRY_BYTES == 160
    assert P.RUNTIME_PRIVATE_BYTES == 49


def test_criterion2_array_capture_footprints():
    # AcceptanceMain.cpp:104-118
    for k, total in zip([1, 2, 3, 4], [617, 1001, 1385, 1769]):
        s, _ = kernel_stack(f"arrays_{k}")
        assert LY.shared_footprint(s) == total == 384 * k + 233


def test_criteria3_to_5_occupancy_tables():
    # AcceptanceMain.cpp:123-222
    k40 = {"vars": [1, 2, 4, 8, 16, 32, 64], "teams": [14, 14, 14, 14, 12, 7, 3],
           "smem": [3262, 3374, 3598, 4046, 4236, 3367, 2211]}
    for i, n in enumerate(k40["vars"]):
        o = OCC.occupancy_for("k40-48k", OCC._footprint(8 * n + 16),
                              OCC.scalars_fixture_regs("k40-48k", n), 128)
        assert (o.actual, o.smem_used) == (k40["teams"][i], k40["smem"][i])
        assert OCC.dynamic_args_bytes(n) == [0, 0, 0, 0, 0, 256, 512][i]
    p100 = {"teams": [16, 16, 16, 16, 12, 7, 3], "smem": [3728, 3856, 4112, 4624, 4236, 3367,
                                                         2211]}
    for i, n in enumerate(k40["vars"]):
        o = OCC.occupancy_for("p100", OCC._footprint(8 * n + 16),
                              OCC.scalars_fixture_regs("p100", n), 128)
        assert (o.actual, o.smem_used) == (p100["teams"][i], p100["smem"][i])
    for i, k in enumerate([1, 2, 3, 4]):
        a = OCC.occupancy_for("k40-16k", OCC._footprint(384 * k + 24), 36, 128)
        assert (a.actual, a.smem_used) == ([14, 14, 11, 9][i], [8638, 14014, 19390, 24766][i])
        b = OCC.occupancy_for("p100", OCC._footprint(384 * k + 24), 30, 128)
        assert (b.actual, b.smem_used) == (17, [10489, 17017, 23545, 30073][i])
    regs = [32, 34, 36, 39, 42, 64, 128, 255, 255]
    published = [98, 106, 116, 128, 140, 226, 482, 994, 2018]
    exact = [True, False, False, True, False, True, True, True, True]
    for i, t in enumerate(OCC.MAX_VARS_TEAM_POINTS):
        assert OCC.max_regs_for_teams("k40-16k", t) == regs[i]
        v = OCC.max_shared_vars("k40-16k", t)
        assert abs(v - published[i]) <= 1
        if exact[i]:
            assert v == published[i]


def test_criterion8_mirror_invariant_every_pipeline():
    # AcceptanceMain.cpp:331-357 (mirror part): TotalShared == TotalLocal
    for p in G.programs():
        for pipe in (P.PIPELINE_DEFAULT, P.PIPELINE_O0, P.PIPELINE_BAD_ORDER):
            out = LU.run_builder(P.lib().ompds_layout_build, p["frame_vars"],
                                 len(p["layouts"]), pipe)
            assert all(g["total_shared"] == g["total_local"] for g in out), p["stem"]


@pytest.mark.gpu
def test_criterion8_allocation_law_on_the_device_runtime():
    # AcceptanceMain.cpp:368-385: 400 rounds, mt19937(20260815), through the
    # __device__ runtime (ompds_rt_replay); results pinned by runtime.json.
    from test_oracle_golden import _replay, check_script
    scripts = [s for s in G.load("runtime") if s["name"].startswith("acceptance_law_")]
    assert len(scripts) == 400
    for s in scripts:
        res, ev, summ = _replay(P.lib().ompds_rt_replay, s)
        check_script(s, res, ev, summ)
        n = s["calls"][1][2]
        assert res[1].addr_kind == (P.ADDR_PREALLOC if n <= 20 else P.ADDR_DYNAMIC)
        assert res[1].live_bytes == (0 if n <= 20 else 8 * n)


def test_criterion7_pass_order_hazard_detected():
    # AcceptanceMain.cpp:281-328 (layout half; the GPU half is
    # test_program.py::test_gpu_reproduces_the_pass_order_miscompile)
    _, bad = kernel_stack("coloring_demo", P.PIPELINE_BAD_ORDER)
    assert bad[0]["overlap_slot"] >= 0
    _, good = kernel_stack("coloring_demo")
    assert all(g["overlap_slot"] < 0 for g in good)
