"""Host logic of the pipelined host-to-host solve (no GPU needed)."""

import pytest

from paper_2311_13862_b200.pipeline import schedule


@pytest.mark.parametrize("count,sub,tail", [(1024, 512, 128), (1024, 256, 64), (64, 32, 8),
                                            (128, 32, 8), (5, 512, 128), (1, 1, 1),
                                            (1000, 300, 75), (7, 2, 1)])
def test_schedule_covers_count_and_tapers(count, sub, tail):
    sizes = schedule(count, sub, tail)
    assert sum(sizes) == count
    assert all(1 <= s <= sub for s in sizes)
    # the un-overlapped last download is at most max(tail, count) ... and never larger than the first
    assert sizes[-1] <= max(tail, min(count, sub))
    assert sizes[-1] <= sizes[0]
