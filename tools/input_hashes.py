"""SHA-256 of every BASELINE config's generated inputs ("the same bytes go to the
oracle and, via H2D, to the GPU; record a hash of each").  Column-major FP64 bytes of A (lda = m)
and Z (ldz = m) as gen/ produces them, plus the tridiagonal workload's d, e, Z.
    python tools/input_hashes.py [configs, e.g. 0,1,4] > profiles/r01_input_hashes.txt"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(memoryview(a).cast("B")).hexdigest()


cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3,4").split(",")]
for k in cfgs:
    p = gen.config(k)
    print(f"configs[{k}] m={p.m} n={p.n}  A {sha(p.A)}  Z {sha(p.Z)}", flush=True)
    del p
w = gen.witness()
print(f"witness m={w.m} n={w.n}  A {sha(w.A)}  Z {sha(w.Z)}")
for key in gen.TRIDIAG_CONFIGS:
    d, e, p = gen.tridiag_config(key)
    print(f"tridiag {key} m={p.m} n={p.n}  d {sha(d)}  e {sha(e)}  Z {sha(p.Z)}")
