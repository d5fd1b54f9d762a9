"""Host-side page allocator of PagedKVCache (no kernel launches): pages are
mapped on demand, scattered placement is a permutation, release returns
pages, and capacity / pool exhaustion raise CapacityError."""

import numpy as np
import pytest

import paper_2505_14884_b200 as pb


def test_allocator_maps_and_releases_pages():
    pc = pb.PagedKVCache(3, 2, 100, 128, page_rows=32, pool_pages=10, device="cpu", seed=4)
    assert pc.capacity == 128 and pc.max_pages == 4
    pc.reserve(0, 33)
    assert (pc.host_table[0, :2] >= 0).all() and (pc.host_table[0, 2:] < 0).all()
    assert pc.block_table[0, :2].tolist() == pc.host_table[0, :2].tolist()
    pc.reserve(0, 64)  # already mapped: no new pages
    assert (pc.host_table[0] >= 0).sum() == 2
    pc.reserve(1, 128)
    pc.reserve(2, 1)
    used = pc.host_table[pc.host_table >= 0]
    assert len(set(used.tolist())) == len(used) == 7
    runs = list(pc._page_rows_of(0, 10, 40))
    assert [(o, r0, r1) for _, o, r0, r1 in runs] == [(10, 10, 32), (0, 32, 40)]
    pc.release(1)
    assert (pc.host_table[1] < 0).all() and len(pc._free) == 10 - 3
    with pytest.raises(pb.CapacityError):
        pc.reserve(0, 129)
    pc.reserve(1, 128)
    pc.reserve(2, 128)  # 2 + 4 + 4 = 10 pages: the whole pool
    with pytest.raises(pb.CapacityError):
        pc.reserve(0, 100)


def test_page_rows_must_be_tile_multiple():
    with pytest.raises(ValueError):
        pb.PagedKVCache(1, 1, 64, 128, page_rows=16, device="cpu")
    pb.PagedKVCache(1, 1, 512, 32, page_rows=128, device="cpu")  # tile = 4096 / 32 = 128 rows
    with pytest.raises(ValueError):
        pb.PagedKVCache(1, 1, 512, 32, page_rows=64, device="cpu")
    assert np.array_equal(pb.PagedKVCache(2, 1, 64, 128, page_rows=32, device="cpu").host_table, -np.ones((2, 2)))
