"""Paper Table 3 (§5.3): the sparse-matrix CPU method with an incomplete Cholesky
preconditioner (drop tolerance 1e-3), one core, on the §5.1 laminate workload (50 CN steps of
dt = 0.01, rtol 1e-6, f = 1 on x3 = 0; C = (30s, 30s, 10s), s = 1..6), next to the paper's
numbers and this repository's B200 runs of the same workload (profiles/r01_table2_laminate.jsonl).
Total time = assembly (the oracle's element scatter into CSR, from precomputed element matrices
as the paper's CPU code) + factorisation + 50 solves, as the paper counts it.

  python tools/ic_comparator.py [s_max] [elem]   (elem 1 = the paper's 6 tets/voxel, 0 = Q1)"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import comparator  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402

PAPER = {1: (0.2, 39), 2: (1.6, 47), 3: (6.2, 54), 4: (16, 56), 5: (37, 62), 6: (67, 67)}   # (total s, iters)


def main():
    smax = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    elem = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    for s in range(1, smax + 1):
        p = synth.laminate(s)
        t0 = time.perf_counter()
        o, F = oracle.problem_oracle(p, elem=elem)
        A = o.csr(p.theta * p.dt, 1.0)
        Lop = o.csr(-(1 - p.theta) * p.dt, 1.0)
        t1 = time.perf_counter()
        f = comparator.ICFactor(A, droptol=1e-3)
        t2 = time.perf_counter()
        u, iters, rc = f.simulate(Lop, F, p.dt, p.nsteps, p.u0, tol=p.rtol)
        t3 = time.perf_counter()
        tot = t3 - t0
        r = {"s": s, "dofs": p.grid.n_nodes, "element": "6 P1 tets / voxel" if elem == 1 else "Q1 hex",
             "rc": rc, "total_iters": int(iters.sum()), "total_s": round(tot, 3),
             "assembly_s": round(t1 - t0, 3), "factor_s": round(t2 - t1, 3), "solve_s": round(t3 - t2, 3),
             "s_per_iter_effective": round(tot / max(1, int(iters.sum())), 5),
             "nnz_A_lower": int((A.nnz + A.shape[0]) // 2), "nnz_L": f.nnz,
             "paper_total_s": PAPER[s][0], "paper_total_iters": PAPER[s][1],
             "host": "1 core (single-threaded C), " + os.uname().nodename}
        print(json.dumps(r), flush=True)
        del o, A, Lop, f


if __name__ == "__main__":
    main()
