"""Reorder inputs that force rejected swaps (test infrastructure).

A rejected swap needs two adjacent diagonal blocks whose Sylvester system is
(numerically) singular, i.e. a shared eigenvalue (reference kernels.cpp:539-540:
rcond < eps^(3/4)).  1x1 <-> 1x1 swaps never reject (Givens, kernels.cpp:515-527)
and a real eigenvalue never equals a complex pair, so every case plants
"twins": an UNSELECTED standardized 2x2 block [[a, b], [-b, a]] and, somewhere
below it, a SELECTED block with exactly the same (a, b).  When the selected
twin reaches its unselected twin the swap is rejected in the reference and in
the GPU window kernel alike (the gap between the twins' eigenvalues stays at
rounding level, rcond ~ 1e-15 << eps^(3/4) = 1.8e-12), the block is recorded
in rejected_blocks and deselected, and later movers stack below it
(reorder.cpp:183-187, 385-391).

The rest of the spectrum is well separated (reals on a grid, pairs with
distinct real parts), the strictly upper fill is uniform [-1, 1) from a
seeded numpy generator.
"""
from __future__ import annotations

import numpy as np


def build(blocks, seed):
    """blocks: list of ("r", lam) or ("c", a, b); returns (S column-major, sizes)."""
    n = sum(1 if b[0] == "r" else 2 for b in blocks)
    rng = np.random.default_rng(seed)
    s = np.triu(rng.uniform(-1.0, 1.0, (n, n)), 1)
    sizes = []
    r = 0
    for b in blocks:
        if b[0] == "r":
            s[r, r] = b[1]
            sizes.append(1)
            r += 1
        else:
            _, a, bb = b
            s[r, r] = s[r + 1, r + 1] = a
            s[r, r + 1] = bb
            s[r + 1, r] = -bb
            sizes.append(2)
            r += 2
    return np.asfortranarray(s), np.array(sizes, dtype=np.uint8)


def case(name):
    """Named rejection scenarios -> (S, sizes, flags, ws)."""
    rng = np.random.default_rng(sum(map(ord, name)))
    if name == "window":
        # one window: [.., twin(unsel), reals, twin(sel), reals(sel)], ws 32
        bl, fl = [], []
        for k in range(4):
            bl.append(("r", -9.0 + k)); fl.append(False)
        bl.append(("c", 0.25, 1.5)); fl.append(False)             # unselected twin
        for k in range(3):
            bl.append(("r", -4.5 + k)); fl.append(k == 1)
        bl.append(("c", 0.25, 1.5)); fl.append(True)              # selected twin
        for k in range(4):
            bl.append(("r", 3.0 + k)); fl.append(k % 2 == 0)
        bl.append(("c", -2.0, 0.5)); fl.append(True)
        return (*build(bl, 11), np.array(fl, dtype=np.uint8), 32)
    if name in ("multigroup", "midchain", "dense", "wide"):
        n_target = {"multigroup": 400, "midchain": 300, "dense": 260, "wide": 1100}[name]
        ws = {"multigroup": 64, "midchain": 24, "dense": 32, "wide": 64}[name]
        ntw = {"multigroup": 3, "midchain": 2, "dense": 5, "wide": 6}[name]
        bl, fl = [], []
        reals = iter(np.linspace(-10.0, 10.0, n_target))
        pair_re = iter(np.linspace(-9.7, 9.7, n_target))
        rows = 0
        twins = [(round(0.5 + 0.37 * k, 6), 2.0 + 0.5 * k) for k in range(ntw)]
        # rows where each twin pair is planted (unselected above, selected below)
        if name == "midchain":
            # the selected twin climbs through several windows before it meets
            # its twin: the stuck event happens in the middle of the chain
            plant = [(40, 200), (90, 260)]
        elif name == "dense":
            plant = [(10 + 45 * k, 30 + 45 * k) for k in range(ntw)]
        elif name == "wide":  # twins on both sides of the slab boundaries of 2-4 ranks
            plant = [(100 + 170 * k, 190 + 170 * k) for k in range(ntw)]
        else:
            plant = [(60 + 110 * k, 100 + 110 * k) for k in range(ntw)]
        pending = sorted([(p[0], 0, k) for k, p in enumerate(plant)] + [(p[1], 1, k) for k, p in enumerate(plant)])
        while rows < n_target:
            if pending and rows >= pending[0][0]:
                _, sel, k = pending.pop(0)
                bl.append(("c", twins[k][0], twins[k][1]))
                fl.append(bool(sel))
                rows += 2
                continue
            if rng.random() < 0.4 and rows + 2 <= n_target:
                bl.append(("c", float(next(pair_re)), float(1 + 2 * rng.integers(0, 3))))
                rows += 2
            else:
                bl.append(("r", float(next(reals))))
                rows += 1
            fl.append(bool(rng.random() < 0.35))
        return (*build(bl, 7 + ntw), np.array(fl, dtype=np.uint8), ws)
    raise KeyError(name)


NAMES = ("window", "multigroup", "midchain", "dense")


def block_eigs(S, sizes):
    """Eigenvalue pair(s) of each diagonal block of the INPUT (as read off)."""
    out = []
    r = 0
    for sz in sizes:
        if sz == 1:
            out.append(complex(S[r, r]))
        else:
            a = S[r, r]
            im = np.sqrt(abs(S[r, r + 1])) * np.sqrt(abs(S[r + 1, r]))
            out.append(complex(a, im))
        r += int(sz)
    return out


def predicted_eigs(S_in, sizes, perm):
    """Eigenvalues read off position by position if block i ended at slot perm[i]."""
    be = block_eigs(S_in, sizes)
    nb = len(sizes)
    slot_blk = np.empty(nb, dtype=np.int64)
    slot_blk[np.asarray(perm, dtype=np.int64)] = np.arange(nb)
    ev = []
    for b in slot_blk:
        e = be[b]
        ev.extend([e] if sizes[b] == 1 else [complex(e.real, e.imag), complex(e.real, -e.imag)])
    return np.array(ev)


def consistent(S_in, sizes, perm, S_out, read_eigenvalues, tol=1e-8):
    """Does the result's permutation describe its matrix? (the reference's
    bookkeeping can diverge after a rejection: SURVEY 8c 'latent caveat')."""
    if sorted(np.asarray(perm).tolist()) != list(range(len(sizes))):
        return False
    want = predicted_eigs(S_in, sizes, perm)
    got = read_eigenvalues(S_out)
    if len(got) != len(want):
        return False
    return bool(np.all(np.abs(got - want) <= tol * np.maximum(1.0, np.abs(want))))


def twins(S, sizes, flags):
    """(unselected twin, selected twin) block indices of a case, top to bottom."""
    be = block_eigs(S, sizes)
    out = []
    for j in range(len(sizes)):
        if sizes[j] != 2 or not flags[j]:
            continue
        for i in range(j - 1, -1, -1):
            if sizes[i] == 2 and not flags[i] and be[i] == be[j]:
                out.append((i, j))
                break
    return out


def predicted_permutation(S, sizes, flags):
    """The arrangement the reference's semantics produce when exactly the
    selected twins are rejected: selected (non-rejected) blocks lead in their
    original order; behind them the unselected blocks in original order, each
    rejected twin directly below its unselected twin (it stops there,
    reorder.cpp:183-187, and is deselected, :385-391; blocks moving past it
    later keep the relative order of everything they pass)."""
    tw = twins(S, sizes, flags)
    rejected = {j for _, j in tw}
    after = {i: j for i, j in tw}
    order = [b for b in range(len(sizes)) if flags[b] and b not in rejected]
    for b in range(len(sizes)):
        if not flags[b]:
            order.append(b)
            if b in after:
                order.append(after[b])
    perm = np.empty(len(sizes), dtype=np.int64)
    perm[np.asarray(order)] = np.arange(len(sizes))
    return perm, sorted(rejected)


# cases whose reference run is well defined (it terminates and its block
# bookkeeping describes its matrix); on the others the reference livelocks
# after the mid-chain rejection (see tests/test_rejection.py)
REF_WELL_DEFINED = ("window", "dense")
REF_LIVELOCKS = ("multigroup", "midchain")
