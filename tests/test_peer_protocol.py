"""Model check of the peer-memory transport's step protocol (include/castfem_b200.h,
cf_comm_create_peer; csrc/cf_api.cu launch_pack_peer / peer_wait_payload / peer_allreduce).

Each rank's stream runs, per step k = 1, 2, ...:
  PACK(k)    store this rank's payload into every neighbour's window, parity k & 1, then raise
             flag[neighbour][me] = k (the stores are ordered before the flag: system-scope fence
             + release);
  WAIT(k)    the stream holds until flag[me][q] >= k for every neighbour q (cuStreamWaitValue32);
  UPDATE(k)  read every neighbour's payload from the own window, parity k & 1.
Ranks run at arbitrary relative speeds. The claim (two parities suffice, no acknowledgement):
UPDATE(k) always reads the payloads of step k. The model executes the ranks' operations one
memory access at a time under a seeded random scheduler; with ONE buffer instead of two the same
scheduler finds an overwrite, so the check has teeth. The scalar all-reduce follows the same
pattern with every rank as a neighbour.
"""
import random

import pytest


def _ops(rank, nbrs, steps):
    """The stream of one rank as a list of atomic operations."""
    ops = []
    for k in range(1, steps + 1):
        for q in nbrs:
            ops.append(("store", q, k))
        for q in nbrs:  # flags after every store of the kernel (last-CTA ticket)
            ops.append(("flag", q, k))
        ops.append(("wait", None, k))
        for q in nbrs:
            ops.append(("read", q, k))
    return ops


def _simulate(nbr, steps, parities, seed):
    R = len(nbr)
    rng = random.Random(seed)
    buf = [[[None] * parities for _ in range(R)] for _ in range(R)]  # buf[owner][sender][parity]
    flag = [[0] * R for _ in range(R)]                               # flag[owner][sender]
    prog = [_ops(r, nbr[r], steps) for r in range(R)]
    pc = [0] * R
    while True:
        runnable = []
        for r in range(R):
            if pc[r] == len(prog[r]):
                continue
            op, q, k = prog[r][pc[r]]
            if op == "wait" and any(flag[r][s] < k for s in nbr[r]):
                continue
            runnable.append(r)
        if not runnable:
            if all(pc[r] == len(prog[r]) for r in range(R)):
                return None
            return "deadlock"
        r = rng.choice(runnable)
        op, q, k = prog[r][pc[r]]
        pc[r] += 1
        if op == "store":
            buf[q][r][k % parities] = (r, k)
        elif op == "flag":
            flag[q][r] = k
        elif op == "read":
            if buf[r][q][k % parities] != (q, k):
                return f"rank {r} step {k}: read {buf[r][q][k % parities]} from {q}"


TOPOLOGIES = {
    "pair": [[1], [0]],
    "chain4": [[1], [0, 2], [1, 3], [2]],
    "ring5": [[(r - 1) % 5, (r + 1) % 5] for r in range(5)],
    "complete4": [[q for q in range(4) if q != r] for r in range(4)],   # = the scalar all-reduce
    "cube8": [[r ^ 1, r ^ 2, r ^ 4] for r in range(8)],                 # RCB of a box into 8
}


@pytest.mark.parametrize("name", sorted(TOPOLOGIES))
def test_two_parities_suffice(name):
    for seed in range(300):
        assert _simulate(TOPOLOGIES[name], steps=6, parities=2, seed=seed) is None, (name, seed)


@pytest.mark.parametrize("name", ["pair", "chain4", "complete4"])
def test_one_buffer_is_caught(name):
    found = [s for s in range(300) if _simulate(TOPOLOGIES[name], steps=6, parities=1, seed=s) not in (None,)]
    assert found, "the scheduler never produced the overwrite a single buffer allows"
