"""Implicit left-balanced tree arithmetic (host side).

Same public names and domain checks as the reference module
/root/reference/pkg/src/lbkd/treemath.py:21-140, so code written against
``lbkd.treemath`` keeps working.  The device kernels carry their own copy
of this arithmetic (csrc/common.cuh).
"""

from __future__ import annotations

MAX_NODES = 2**31 - 1  # 32-bit tags (treemath.py:16-18)


def _need_node(i: int) -> None:
    if i < 0:
        raise ValueError("negative node index")


def parent(i: int) -> int:
    if i < 1:
        raise ValueError("node 0 is the root and has no parent")
    return (i - 1) >> 1


def left_child(i: int) -> int:
    _need_node(i)
    return 2 * i + 1


def right_child(i: int) -> int:
    _need_node(i)
    return 2 * i + 2


def level(i: int) -> int:
    _need_node(i)
    return (i + 1).bit_length() - 1


def num_levels(n: int) -> int:
    if n < 1:
        raise ValueError("tree must have at least one node")
    return n.bit_length()


def full_tree_size(levels: int) -> int:
    if levels < 0:
        raise ValueError("negative level count")
    return (1 << levels) - 1


def _in_tree(s: int, n: int) -> None:
    if not 0 <= s < n:
        raise ValueError("node index out of range")


def leftmost_bottom_slot(s: int, n: int) -> int:
    _in_tree(s, n)
    return ((s + 1) << (num_levels(n) - level(s) - 1)) - 1


def subtree_size(s: int, n: int) -> int:
    _in_tree(s, n)
    sh = num_levels(n) - level(s) - 1
    width = 1 << sh
    present = n - leftmost_bottom_slot(s, n)
    return width - 1 + min(max(present, 0), width)


def num_left_siblings(s: int) -> int:
    _need_node(s)
    return s - full_tree_size(level(s))


def segment_begin(s: int, n: int) -> int:
    _in_tree(s, n)
    lv = level(s)
    sh = num_levels(n) - lv - 1
    top = full_tree_size(lv)
    left = s - top
    bottom_total = n - full_tree_size(num_levels(n) - 1)
    return top + left * ((1 << sh) - 1) + min(left << sh, bottom_total)


def pivot_pos(s: int, n: int) -> int:
    c = 2 * s + 1
    b = segment_begin(s, n)
    return b + subtree_size(c, n) if c < n else b


# --- working-array helpers used to rebuild BuildRecorder snapshots ---------

def segment_sizes(n: int, l: int):
    """Sizes of the 2^l level-l segments (the not-yet-final points)."""
    L = num_levels(n)
    sh = L - l - 1
    bottom = n - full_tree_size(L - 1)
    w = 1 << sh
    return [w - 1 + min(max(bottom - (j << sh), 0), w) for j in range(1 << l)]
