"""Exact host replicas of NumPy's pairwise summation tree.

The reference engine sums every consensus segment with
``np.add.reduceat`` (``fgadmm/engine.py:279``) and every variable's edge
weights with ``np.add.reduce`` (``fgadmm/graph.py:219``).  Both run
NumPy's fixed pairwise tree (8 accumulators, leaves of <= 128, halving
splits rounded down to a multiple of 8), so the tree shape depends only
on the segment length.  This module

* enumerates that tree (leaves + combine order) for the device plan,
  which replays it bit-exactly on the GPU, and
* evaluates grouped segment sums on the host for the graph layer
  (``z_weights``) without a Python loop per variable.

Used by the host plan builder; it does no per-iteration work.
"""

from __future__ import annotations

import numpy as np

PW_BLOCK = 128   # NumPy PW_BLOCKSIZE
PW_UNROLL = 8    # NumPy's accumulator count


def pairwise_leaves(n):
    """Leaves of NumPy's pairwise tree over ``n`` items, in order.

    Returns a list of ``(start, length)``; every leaf has
    ``length <= 128``.  ``n == 0`` yields no leaves.
    """
    out = []
    stack = [(0, int(n))]
    while stack:
        s, m = stack.pop()
        if m <= PW_BLOCK:
            if m > 0:
                out.append((s, m))
            continue
        h = m // 2
        h -= h % PW_UNROLL
        # right pushed first so the left half is expanded first
        stack.append((s + h, m - h))
        stack.append((s, h))
    return out


def pairwise_split(n):
    """Split point NumPy uses for a node of ``n > 128`` items."""
    h = n // 2
    return h - h % PW_UNROLL


def leaf_sum(a):
    """NumPy's leaf kernel (``n <= 128``) restated with scalar adds."""
    n = len(a)
    if n < PW_UNROLL:
        res = 0.0
        for v in a:
            res += float(v)
        return res
    r = [float(v) for v in a[:PW_UNROLL]]
    i = PW_UNROLL
    top = n - n % PW_UNROLL
    while i < top:
        for j in range(PW_UNROLL):
            r[j] += float(a[i + j])
        i += PW_UNROLL
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < n:
        res += float(a[i])
        i += 1
    return res


def pairwise_sum(a):
    """Scalar restatement of NumPy's pairwise sum (test helper)."""
    n = len(a)
    if n <= PW_BLOCK:
        return leaf_sum(a)
    h = pairwise_split(n)
    return pairwise_sum(a[:h]) + pairwise_sum(a[h:])


def grouped_reduce(values, starts, lengths):
    """Per-segment ``np.add.reduce`` with NumPy's exact rounding.

    ``values[starts[i]:starts[i]+lengths[i]]`` is segment ``i``.  Short
    segments (< 8 items, where the tree is a left fold from 0.0) are
    summed column-wise in one vectorized pass per length; longer ones
    call ``np.add.reduce`` on the 1-D slice, which is exactly the
    reference's own call (``fgadmm/graph.py:219``).
    """
    values = np.asarray(values, dtype=np.float64)
    starts = np.asarray(starts, dtype=np.int64)
    lengths = np.asarray(lengths, dtype=np.int64)
    out = np.zeros(len(starts), dtype=np.float64)
    for L in np.unique(lengths):
        L = int(L)
        sel = np.nonzero(lengths == L)[0]
        if L == 0:
            continue
        if L < PW_UNROLL:
            acc = np.zeros(len(sel), dtype=np.float64)
            base = starts[sel]
            for j in range(L):
                acc = acc + values[base + j]
            out[sel] = acc
        else:
            for i in sel:
                s = int(starts[i])
                out[i] = float(np.add.reduce(values[s:s + L]))
    return out
