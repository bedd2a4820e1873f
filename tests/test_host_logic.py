"""Host-side logic that needs no GPU: group offsets of row-partitioned runs."""
import pytest

from paper_2212_04540_b200.quantize import row_group_offset


def test_row_group_offset_per_row_and_grouped():
    assert row_group_offset(0, 64, None) == 0
    assert row_group_offset(1000, 64, None) == 1000          # one group per row
    assert row_group_offset(1000, 64, 32) == 2000            # G < d: d/G groups per row
    assert row_group_offset(1000, 64, 128) == 500            # G > d: a group spans 2 rows
    assert row_group_offset(1000, 64, 256) == 250
    with pytest.raises(ValueError):
        row_group_offset(1001, 64, 128)                      # block starts inside a group


def test_partition_layout_choice():
    import numpy as np
    from paper_2212_04540_b200.parallel import RowPartition
    eq = RowPartition(4, 0, np.array([0, 100, 200, 300, 400]), 400)
    assert eq.preferred_layout() == "padded"
    skew = RowPartition(4, 0, np.array([0, 10, 200, 300, 400]), 400)
    assert skew.preferred_layout() == "global"


def test_rows_concat_view_or_copy():
    """The BPR gradients reach the compact scatter without a concatenation
    when they already lie back to back in scatter order (functional._rows_concat);
    any other layout falls back to torch.cat with the same values."""
    import torch
    from paper_2212_04540_b200.functional import _rows_concat
    buf = torch.arange(3 * 5 * 4, dtype=torch.float32).reshape(3, 5, 4)
    v = _rows_concat([buf[0], buf[1], buf[2]], 4)
    assert v.data_ptr() == buf.data_ptr() and torch.equal(v, buf.reshape(-1, 4))
    w = _rows_concat([buf[2], buf[1], buf[0]], 4)
    assert w.data_ptr() != buf.data_ptr() and torch.equal(w, torch.cat([buf[2], buf[1], buf[0]]))
    gap = _rows_concat([buf[0], buf[2]], 4)
    assert torch.equal(gap, torch.cat([buf[0], buf[2]]))
    other = torch.zeros(5, 4)
    assert torch.equal(_rows_concat([buf[0], other], 4), torch.cat([buf[0], other]))


def test_retired_readout_refuses_other_rows():
    """A sum readout whose terms were retired to the batch's rows
    (forward_all(readout_rows=...)) refuses to materialize and refuses a
    gather at other indices (no kernel runs before the check)."""
    import torch
    from paper_2212_04540_b200.tape import LazySumWire, RetiredRows, RetiredSum, TapeUsageError
    idx = torch.arange(4, dtype=torch.int64)
    acc = RetiredSum(torch.zeros(4, 8), idx)
    acc.n_terms = 2
    terms = [RetiredRows(("node", 3), (10, 8), acc), RetiredRows(("node", 6), (10, 8), acc)]
    w = LazySumWire(("node", 9), terms)
    assert w.shape == (10, 8)
    with pytest.raises(TapeUsageError):
        w.value
    with pytest.raises(TapeUsageError):
        w.index_select_rows(torch.arange(4, dtype=torch.int64))     # same values, other tensor
    assert torch.equal(w.index_select_rows(idx), acc.rows)              # all terms retired: the sum itself
    acc.n_terms = 1                                                     # a term missing from the sum
    with pytest.raises(TapeUsageError):
        w.index_select_rows(idx)
