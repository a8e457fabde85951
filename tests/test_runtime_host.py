"""Host-side runtime logic without a GPU: the decode-attention work split
(runtime.decode_chunks) and the piggyback completion tag encoding."""

import pytest

from paper_2603_12831_b200 import runtime
from paper_2603_12831_b200.runtime import decode_chunks, result_tag


def _check_cover(ctxs, chunks, begin):
    """Every row's pages are covered exactly once, in order, by its chunks."""
    assert begin[0] == 0 and len(begin) == len(ctxs) + 1
    for r, c in enumerate(ctxs):
        own = chunks[begin[r]:begin[r + 1]]
        pages = (c + 63) // 64
        assert own[0][2] == 0 and own[-1][3] == pages
        for a, b in zip(own, own[1:]):
            assert a[3] == b[2]
        assert all(ch[0] == r and ch[4] == c for ch in own)


@pytest.mark.parametrize("ctxs", [[701] * 8, [701] * 32, [9001] * 8, [9001], [701] * 8 + [9001] * 2,
                                  [1, 64, 65, 129], [2001] * 4])
def test_decode_chunks_cover_rows(ctxs):
    chunks, begin = decode_chunks(ctxs, 8)
    _check_cover(ctxs, chunks, begin)
    # at most 64 pages per chunk (bounded merge fan-in)
    assert max(c[3] - c[2] for c in chunks) <= 64


def test_decode_chunks_small_batch_keeps_short_rows_whole():
    chunks, _ = decode_chunks([701] * 8, 8)  # 88 page-heads x 8 <= 2048, 11 pages per row
    assert len(chunks) == 8
    chunks, _ = decode_chunks([701] * 32, 8)  # large enough: one wave of <= 296 CTAs
    assert len(chunks) * 8 <= 296
    chunks, _ = decode_chunks([2001] * 4, 8)  # rows of 32 pages are still split
    assert len(chunks) > 4


def test_decode_chunks_without_small_rule(monkeypatch):
    monkeypatch.setattr(runtime, "SMALL_KV_PAGE_HEADS", 0)
    chunks, begin = decode_chunks([701] * 8, 8)
    _check_cover([701] * 8, chunks, begin)
    assert len(chunks) * 8 <= 296 and len(chunks) > 8  # split to fill the wave


def test_result_tag_matches_header_macro():
    # HS_RESULT_TAG(ctx, layer) = (int)(((unsigned)ctx << 8) | layer)
    assert result_tag(5, 1) == (5 << 8) | 1
    assert result_tag(33000, 80) == (33000 << 8) | 80
    assert result_tag(1 << 24, 3) == 3  # wraps like the unsigned 32-bit shift in C
    assert result_tag((1 << 23) + 1, 2) == -(1 << 31) + (1 << 8) + 2  # sign bit set: negative int
