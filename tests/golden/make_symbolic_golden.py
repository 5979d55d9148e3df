"""Write tests/golden/symbolic_<config>.json from the ORACLE only (gen + oracle, no CUDA path).

Each file holds sha256 digests of the oracle's integer symbolic arrays for
one config, so that the CPU test suite can check the fast analyze path bit-exactly on the full
configs without re-running the (slow) oracle symbolic phase every time.
Run:  python tests/golden/make_symbolic_golden.py C1 C2 C3 C4 C5
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402

KEYS = ["post", "parent3", "cc3", "ffirst", "fgroup", "perm_final", "sfirst", "sparent", "rows_ptr", "rows",
        "rel_ptr", "rel_anc", "rel_q0", "rel_off", "relind", "parent_final", "cc_final"]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(names):
    for name in names:
        p = gen.make(name)
        o = oracle.Oracle.from_problem(p, keep_L=False)
        s = o.symbolic()
        out = {"config": name, "desc": gen.CONFIGS[name]["desc"], "n": p.n, "nnz_A": p.nnz, "nnz_L": o.nnzL,
               "flops_exact": o.flops, "nfund": o.nfund, "nsuper": o.nsuper, "added": o.added,
               "nmerges": o.nmerges, "sha256": {k: digest(s[k]) for k in KEYS},
               "dtypes": {k: str(s[k].dtype) for k in KEYS},
               "_source": "oracle/ only (tests/golden/make_symbolic_golden.py)"}
        with open(os.path.join(HERE, f"symbolic_{name}.json"), "w") as f:
            json.dump(out, f, indent=1)
        print(name, o.nnzL, o.nsuper, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"])
