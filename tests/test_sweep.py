"""NEXT-4: checkpointed sweeps resume byte-identically; shard states merge to the unsharded state.

CPU tests use a stand-in block evaluator built from the oracle's prime list (values are stand-ins:
the resume/merge logic is what is tested); the GPU test runs the CUDA evaluator."""
import json
import os

import pytest

from paper_2101_11157_b200 import sweep as sw


def _fake_eval(lo, hi, mode, bound):
    import oracle
    ps = oracle.primes(max(lo, 5), hi)
    chk = sum((p * 0x9E3779B97F4A7C15) & ((1 << 64) - 1) for p in ps) & ((1 << 64) - 1)
    hits = [(p, 1) for p in ps if p % 1000 == 7]
    near = [(p, 2, (p % 99) - 49) for p in ps if p % 97 == 3]
    hw = [0] * 2000
    hv = [0] * 2000
    for p in ps:
        hw[p % 2000] += 1
    return len(ps), chk, hits, near, hw, hv


def test_resume_is_byte_identical(tmp_path):
    lo, hi, block = 10 ** 6, 10 ** 6 + 7 * 32768 + 123, 32768
    full = tmp_path / "full.json"
    part = tmp_path / "part.json"
    sw.sweep(lo, hi, 3, block, str(full), evaluate=_fake_eval)
    s = sw.sweep(lo, hi, 3, block, str(part), max_blocks=3, evaluate=_fake_eval)
    assert not s["done"] and s["next_block"] == 3
    s = sw.sweep(lo, hi, 3, block, str(part), max_blocks=2, evaluate=_fake_eval)
    assert s["next_block"] == 5
    s = sw.sweep(lo, hi, 3, block, str(part), evaluate=_fake_eval)
    assert s["done"]
    assert full.read_bytes() == part.read_bytes()
    with pytest.raises(ValueError):
        sw.sweep(lo, hi + 1, 3, block, str(part), evaluate=_fake_eval)


def test_shard_states_merge_to_unsharded(tmp_path):
    lo, hi, block = 3 * 10 ** 6, 3 * 10 ** 6 + 9 * 32768 + 55, 32768
    whole = sw.sweep(lo, hi, 3, block, str(tmp_path / "w.json"), evaluate=_fake_eval)
    parts = [sw.sweep(lo, hi, 3, block, str(tmp_path / f"s{r}.json"), shard=r, nshards=3, evaluate=_fake_eval)
             for r in range(3)]
    m = sw.merge_states(parts)
    for k in ("primes", "checksum", "hits", "near", "hist_w", "hist_v"):
        assert m[k] == whole[k], k
    # the snake interleave covers every block exactly once
    bl = sorted(b for r in range(3) for b in sw.blocks_of(lo, hi, block, r, 3))
    assert bl == sw.blocks_of(lo, hi, block)


@pytest.mark.gpu
def test_gpu_sweep_matches_search(tmp_path, wv):
    """The CUDA evaluator: an interrupted sweep of C1 equals the uninterrupted one byte for byte and
    equals one wv_search over the window (hits, checksum); the near-miss/histogram totals are sane."""
    lo, hi, block = 5, 10 ** 5, 32768
    a = sw.sweep(lo, hi, 3, block, str(tmp_path / "a.json"))
    sw.sweep(lo, hi, 3, block, str(tmp_path / "b.json"), max_blocks=1)
    b = sw.sweep(lo, hi, 3, block, str(tmp_path / "b.json"))
    assert (tmp_path / "a.json").read_bytes() == (tmp_path / "b.json").read_bytes()
    hits, res, chk = wv.search_shard(lo, hi, 3, 0, 1, 0)
    assert a["checksum"] == str(chk) and a["primes"] == len(res) == 9590
    assert [[str(int(h["p"])), int(h["flags"])] for h in hits] == a["hits"]
    assert sum(a["hist_w"]) == sum(a["hist_v"]) == 9590


def test_merge_rejects_duplicate_or_missing_shards(tmp_path):
    lo, hi, block = 3 * 10 ** 6, 3 * 10 ** 6 + 5 * 32768, 32768
    parts = [sw.sweep(lo, hi, 3, block, str(tmp_path / f"s{r}.json"), shard=r, nshards=3, evaluate=_fake_eval)
             for r in range(3)]
    with pytest.raises(ValueError):
        sw.merge_states([parts[0], parts[0], parts[1]])
    with pytest.raises(ValueError):
        sw.merge_states(parts[:2])
    sw.merge_states([parts[2], parts[0], parts[1]])      # any order of the complete set


def test_checkpoint_records_partition_and_block_count(tmp_path):
    """A checkpoint names its partition (and format); one written under another partition, or whose
    block count disagrees with this partition's, is refused instead of resumed into the wrong blocks."""
    lo, hi, block = 10 ** 6, 10 ** 6 + 6 * 32768, 32768
    path = tmp_path / "c.json"
    s = sw.sweep(lo, hi, 3, block, str(path), shard=1, nshards=2, max_blocks=1, evaluate=_fake_eval)
    assert s["config"]["partition"] == sw.PARTITION and s["config"]["format"] == sw.FORMAT
    old = json.loads(path.read_text())
    old["config"]["partition"] = "interleave-v1"
    path.write_text(json.dumps(old))
    with pytest.raises(ValueError):
        sw.sweep(lo, hi, 3, block, str(path), shard=1, nshards=2, evaluate=_fake_eval)
    s = sw.new_state(lo, hi, 3, block, 50, 1, 2)
    s["blocks"] += 1
    s["next_block"] = 1
    path.write_text(json.dumps(s))
    with pytest.raises(ValueError):
        sw.sweep(lo, hi, 3, block, str(path), shard=1, nshards=2, evaluate=_fake_eval)


def test_blocks_of_equals_library_partition():
    """sweep.blocks_of (Python) and wv_shard_blocks (the C ABI that wv_search_shard uses) describe the
    same partition, for ragged windows, several block sizes and shard counts (host-only call)."""
    import __graft_entry__ as g
    g.build()
    from paper_2101_11157_b200 import _wv
    import random
    rng = random.Random(4)
    for _ in range(40):
        lo = rng.randrange(5, 10 ** 9)
        block = 1 << rng.randrange(17, 21)
        hi = lo + rng.randrange(1, 70) * block + rng.randrange(0, block)
        n = rng.randrange(1, 9)
        for r in range(n):
            lib_blocks, used = _wv.shard_blocks(lo, hi, r, n, block)
            assert used == block
            assert [tuple(map(int, b)) for b in lib_blocks] == sw.blocks_of(lo, hi, block, r, n), (lo, hi, block, r, n)
