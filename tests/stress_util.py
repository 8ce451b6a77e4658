"""Randomized launches of the config kernels over launch parameters, each
checked against the oracle: values, traps, regions and balanced args-list
allocations.  Used by tests/test_gpu_stress.py (a seeded slice in the GPU
suite) and tools/stress.py (longer runs)."""
import random

import numpy as np
import torch

from oracle import oracle as O
from paper_1711_10413_b200 import regions as RG

COEF = [k / 8 for k in range(1, 9)]


def one_launch(rng: random.Random, it: int):
    """Runs one random launch; returns (ok, description)."""
    kind = rng.choice(["regions", "stream", "shared", "nested"])
    teams = rng.choice([1, 2, 3, 7, 64, 148, 300])
    workers = rng.choice([1, 2, 31, 32, 33, 63, 64, 96, 100, 255, 480, 992])
    kw = dict(prealloc_entries=rng.choice([0, 1, 2, 4, 8, 20, 64]),
              list_allocator=rng.choice([0, 0, 1]))
    log = rng.random() < 0.25 and teams * workers <= 20000
    if log:
        kw["max_events"] = 4 * workers + 64 if kind != "regions" else 16 * (2 * workers + 8)
    if kind == "regions":
        R = rng.choice([1, 2, 5])
        elem = rng.choice([0, 1])
        a = torch.zeros(teams * workers, dtype=torch.float64 if elem else torch.int32,
                        device="cuda")
        out = RG.run_regions(a, teams, workers, R, **kw)
        want = np.zeros(teams * workers, dtype=np.float64 if elem else np.int32)
        O.lib().orc_regions(elem, teams, workers, R, O.ptr(want))
        ok = np.array_equal(a.cpu().numpy(), want)
        exp_regions = R
    elif kind == "stream":
        n = rng.choice([1, 7, 1000, 65537, 1 << 20])
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        RG.fill_uniform(x, 1 + it)
        RG.fill_uniform(y, 2 + it)
        xs, ys = x.cpu().numpy().copy(), y.cpu().numpy().copy()
        out = RG.run_stream(x, y, COEF, teams, workers, **kw)
        O.lib().orc_stream(1, n, O.ptr(xs), O.ptr(ys), O.ptr(np.array(COEF)), 0)
        ok = np.array_equal(y.cpu().numpy().view(np.uint64), ys.view(np.uint64))
        exp_regions = 1
    elif kind == "shared":
        n = rng.choice([1, 255, 4096, 100003])
        a = torch.zeros(n, dtype=torch.float64, device="cuda")
        d = torch.arange(256, dtype=torch.float64, device="cuda") * 3 + 1
        out = RG.run_shared_array(a, teams, workers, d_init=d, **kw)
        ai = np.arange(n)
        ok = np.array_equal(a.cpu().numpy(), (3 * (ai & 255) + 1).astype(np.float64))
        exp_regions = 1
    else:
        R = rng.choice([1, 3])
        elem = rng.choice([0, 1])
        kw.pop("max_events", None)
        a = torch.zeros(teams * workers, dtype=torch.float64 if elem else torch.int32,
                        device="cuda")
        out, _ = RG.run_nested(a, teams, workers, R, **kw)
        want = np.zeros(teams * workers, dtype=np.float64 if elem else np.int32)
        O.lib().orc_nested(elem, teams, workers, R, O.ptr(want))
        ok = np.array_equal(a.cpu().numpy(), want)
        exp_regions = R
    st = out.team_stats()
    traps = {s.trap for s in st}
    ok = ok and traps == {0} and all(s.regions == exp_regions and
                                     s.dynamic_allocs == s.dynamic_frees for s in st)
    return ok, (it, kind, teams, workers, kw, traps)


def run(seed: int, iterations: int):
    """Returns the descriptions of the failing launches (empty: all exact)."""
    rng = random.Random(seed)
    return [desc for it in range(iterations) for ok, desc in [one_launch(rng, it)] if not ok]
