"""Discrete-event simulator of one GPipe iteration (test infrastructure).

PAPER.md:122-129 (Sec. 3.2, Fig. 3, Eq. 2) models the time per iteration of
a GPipe-style schedule as

    tpi = sum_i p_i + sum_j o_j + (c - 1) * max(P u O)

where p_i is stage i's forward + backward time per micro-batch and o_j the
forward + backward transfer time across cut j.  This module does not use
that formula: it replays the schedule event by event and returns the
makespan, so tests can check Eq. 2 (and the oracle's objective, which
evaluates it) against an independent model of the same schedule.

Schedule (GPipe with a flush): the pipeline is a chain of
"servers" -- stage 1, link 1, stage 2, ..., stage deg.  All c micro-batches
run forward through the chain in order; a server starts micro-batch m when it
has finished micro-batch m-1 and the previous server has finished micro-batch
m.  The backward pass runs through the chain in reverse, starting at the last
stage once it has finished its last forward; a server starts the backward of
a micro-batch when it has finished the previous backward, the next server has
finished that micro-batch's backward, and (flush) it has finished all of its
forwards.  No two operations overlap on one server.
"""
from __future__ import annotations


def simulate(fwd, bwd, c):
    """Makespan of one GPipe iteration.

    fwd[s], bwd[s]: per-micro-batch forward / backward time of server s in
    pipeline order (stages and links interleaved); c: micro-batches.
    Returns (makespan, per-server event log) with exact (integer or
    Fraction) arithmetic if the inputs are exact.
    """
    K = len(fwd)
    assert K == len(bwd) and K >= 1 and c >= 1
    end_f = [[0] * c for _ in range(K)]
    log = [[] for _ in range(K)]
    for m in range(c):
        for s in range(K):
            ready = end_f[s - 1][m] if s > 0 else 0
            free = end_f[s][m - 1] if m > 0 else 0
            start = max(ready, free)
            end_f[s][m] = start + fwd[s]
            log[s].append(("F", m, start, end_f[s][m]))
    end_b = [[0] * c for _ in range(K)]
    for m in range(c):  # backward micro-batch order: c-1, ..., 0 (any order: equal times)
        mb = c - 1 - m
        for s in range(K - 1, -1, -1):
            ready = end_b[s + 1][mb] if s < K - 1 else 0
            prev = end_b[s][c - m] if m > 0 else 0  # the previous backward on this server
            flush = end_f[s][c - 1]
            start = max(ready, prev, flush)
            end_b[s][mb] = start + bwd[s]
            log[s].append(("B", mb, start, end_b[s][mb]))
    return end_b[0][0], log


def no_overlap(log):
    """Every server runs one operation at a time."""
    for ops in log:
        iv = sorted((a, b) for _, _, a, b in ops)
        for (a0, b0), (a1, b1) in zip(iv, iv[1:]):
            if a1 < b0:
                return False
    return True


def eq2(p, o, c):
    """Eq. 2 written out -- for the tests' comparison only."""
    return sum(p) + sum(o) + (c - 1) * max(list(p) + list(o))


def servers(stage_fwd, stage_bwd, link_fwd, link_bwd):
    """Interleave stages and links into the server chain."""
    f, b = [], []
    for i in range(len(stage_fwd)):
        f.append(stage_fwd[i])
        b.append(stage_bwd[i])
        if i < len(link_fwd):
            f.append(link_fwd[i])
            b.append(link_bwd[i])
    return f, b
