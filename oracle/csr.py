"""Oracle: batch construction and batch transposes (brute force).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* The stream is the dataset in a fixed order (reading R10: identity, or one
  seeded permutation for the whole run); batch j of a mega-batch takes the
  next ``rows`` samples of the stream ("batches are dispatched
  one-by-one").  Batch CSR is rebased to 0.
* Transposes (not in the paper; D11 of SURVEY.md): the nnz of a batch sorted
  by (feature, row) and the labels sorted by (label, row).  The brute force
  here sorts explicit (key, row) pairs with Python's sort -- a different
  algorithm from any device counting sort.
"""
from __future__ import annotations

import numpy as np


def stream_ids(pos, rows, n, order=None):
    """Sample ids of stream positions pos .. pos+rows-1 (wrapping per data
    epoch).  order=None is the identity order."""
    p = (np.arange(rows, dtype=np.int64) + int(pos)) % int(n)
    return p if order is None else np.asarray(order, np.int64)[p]


def batch_csr(dataset, ids):
    """Rebased CSR of the given sample ids: (row_ptr, col, val, lab_ptr, lab)."""
    row_ptr = [0]; col = []; val = []; lab_ptr = [0]; lab = []
    for i in ids:
        s, e = int(dataset.row_ptr[i]), int(dataset.row_ptr[i + 1])
        col.extend(int(x) for x in dataset.col[s:e]); val.extend(dataset.val[s:e].tolist())
        row_ptr.append(len(col))
        s, e = int(dataset.lab_ptr[i]), int(dataset.lab_ptr[i + 1])
        lab.extend(int(x) for x in dataset.lab[s:e]); lab_ptr.append(len(lab))
    return (np.array(row_ptr, np.int64), np.array(col, np.int32), np.array(val, np.float32),
            np.array(lab_ptr, np.int64), np.array(lab, np.int32))


def transpose(ptr, idx, val=None):
    """Sort the entries (row r, key idx[j]) by (key, r).

    Returns (seg_key, seg_ptr, seg_row, seg_val): unique keys ascending, segment
    boundaries, rows (ascending inside a segment) and values in that order."""
    entries = []
    for r in range(len(ptr) - 1):
        for j in range(int(ptr[r]), int(ptr[r + 1])):
            entries.append((int(idx[j]), r, j))
    entries.sort()
    keys = []; seg_ptr = [0]; rows = []; vals = []
    for k, r, j in entries:
        if not keys or keys[-1] != k:
            if keys:
                seg_ptr.append(len(rows))
            keys.append(k)
        rows.append(r)
        if val is not None:
            vals.append(val[j])
    seg_ptr.append(len(rows))
    if not keys:
        seg_ptr = [0]
    return (np.array(keys, np.int32), np.array(seg_ptr, np.int32), np.array(rows, np.int32),
            np.array(vals, np.float32) if val is not None else None)
