"""Completion tags of the piggyback result mailbox (the device-checked gate of
Attention Piggybacking): a merged row whose host result was not published
with the expected tag must surface as the reference's IntegrityFault
(pkg/src/hybridserve/errors.py:12-18), and a published one must pass."""

import pytest

from paper_2603_12831_b200.errors import IntegrityFault
from paper_2603_12831_b200.models import TRANSFORMERS


def _iteration(ctx, cfg, tag):
    # one decode row (slot 0, position 5) and, at layer 1, one merged chain
    # (slot 3) carrying `tag`
    ctx.iter_begin([0], [5], [-1], 1, [(0, 0, 0, 1, 6)], [0, 1], [], [0])
    for layer in range(1, cfg.n_layers + 1):
        merge = layer == 1
        ctx.layer(layer, [], [], [3] if merge else [], [], [], [tag] if merge else [])
    return ctx.iter_end()


@pytest.mark.gpu
def test_merge_of_unpublished_result_is_integrity_fault(cuda):
    from paper_2603_12831_b200.runtime import HsContext, RuntimeConfig, result_tag

    cfg = TRANSFORMERS["tiny"]
    ctx = HsContext(cfg, RuntimeConfig(max_rows=64, max_slots=8, kv_pages=16, max_pages_per_req=4,
                                       max_pos=256, max_chunks=64, cpu_threads=1,
                                       host_kv_bytes=8 << 20))
    ctx.init_weights(0)
    ctx.set_page_table(0, [0])
    ctx.host_kv_reserve(3, 64)
    with pytest.raises(IntegrityFault):
        _iteration(ctx, cfg, result_tag(5, 1))  # nothing published for slot 3 yet
    ctx.cpu_attend([3], [1], [5])  # the worker publishes result_tag(5, 1)
    assert len(_iteration(ctx, cfg, result_tag(5, 1))) == 1
    with pytest.raises(IntegrityFault):
        _iteration(ctx, cfg, result_tag(6, 1))  # a stale result (previous token)
    ctx.close()
