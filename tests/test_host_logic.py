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
