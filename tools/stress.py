"""Randomized stress of the config kernels over launch parameters, checked
against the oracle (validation tool; the GPU suite runs a seeded slice of the
same generator, tests/test_gpu_stress.py):

    python tools/stress.py [seed] [iterations]
"""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import stress_util  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 7
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
fails = stress_util.run(seed, iters)
for f in fails:
    print("FAIL", f)
print(f"stress: {iters - len(fails)}/{iters} launches exact")
sys.exit(1 if fails else 0)
