"""Long sweeps with checkpoint / resume (SPEC scanner S:L471-474, L499-507).

A sweep walks [lo, hi) in fixed blocks, in order, and after every block writes a
JSON checkpoint atomically (write to a temp file, then rename).  The state holds
the configuration (and its digest), the next block, and the accumulated outputs:
prime count, order-independent checksum (reading R6), hits, near misses
(|<r>_p| < bound) and the two 2000-bin histograms of <r>_p / p.
Running the same sweep again resumes at `next_block`; the final checkpoint is
byte-identical whether or not the run was interrupted (all lists sorted, keys
sorted, integers as decimal strings where they can exceed 2^53).

With N GPUs, rank r sweeps the blocks of shard r (same snake interleave as
wv_search_shard) into its own state file; merge_states() combines them into the
state an unsharded sweep produces (same checksum, hits, near misses, histograms).

The per-block work is `evaluate(lo, hi, mode, near_bound)`; the default runs the
CUDA path (DeviceSearch + wv_near_misses_device).  Tests substitute a CPU stand-in
to exercise the resume logic without a GPU.
"""
from __future__ import annotations

import hashlib
import json
import os

M64 = (1 << 64) - 1
# Block order of a shard.  Part of the configuration (and so of the digest): a checkpoint written
# under another partition must not resume into this one's block list.
PARTITION = "snake-top-v2"
FORMAT = 2


def _digest(cfg: dict) -> str:
    return hashlib.sha256(json.dumps(cfg, sort_keys=True).encode()).hexdigest()[:16]


def gpu_block_evaluator(lo: int, hi: int, mode: int, near_bound: int):
    """One block on the current CUDA device: (n_primes, checksum, hits, near, hist_w, hist_v)."""
    from . import _wv
    ds = _wv.DeviceSearch(lo, hi, mode).run()
    near, hw, hv = ds.near_misses(near_bound)
    hits = [(int(h["p"]), int(h["flags"])) for h in ds.hits_np()]
    nm = [(int(x["p"]), int(x["test"]), int(x["symres"])) for x in near]
    return ds.n_primes, ds.checksum_int(), hits, nm, [int(x) for x in hw], [int(x) for x in hv]


def blocks_of(lo: int, hi: int, block: int, shard: int = 0, nshards: int = 1):
    """This shard's blocks in sweep order (snake interleave; see include/wv.h wv_search_shard)."""
    nb = (hi - lo + block - 1) // block
    pad = (-nb) % nshards          # rounds aligned to the top of the window (virtual empty blocks below 0)
    out = []
    for j in range((nb + pad) // nshards):
        b = j * nshards + ((nshards - 1 - shard) if (j & 1) else shard) - pad
        if b >= 0:
            out.append((lo + b * block, min(lo + (b + 1) * block, hi)))
    return out


def new_state(lo, hi, mode, block, near_bound, shard=0, nshards=1) -> dict:
    cfg = dict(lo=str(lo), hi=str(hi), mode=mode, block=str(block), near_bound=near_bound, shard=shard,
               nshards=nshards, hist_bins=2000, partition=PARTITION, format=FORMAT)
    return dict(config=cfg, digest=_digest(cfg), next_block=0, blocks=len(blocks_of(lo, hi, block, shard, nshards)),
                primes=0, checksum="0", hits=[], near=[], hist_w=[0] * 2000, hist_v=[0] * 2000, done=False)


def _write(path: str, state: dict):
    tmp = f"{path}.tmp{os.getpid()}"
    with open(tmp, "w") as f:
        json.dump(state, f, sort_keys=True, separators=(",", ":"))
        f.write("\n")
    os.replace(tmp, path)


def sweep(lo: int, hi: int, mode: int, block: int, state_path: str, near_bound: int = 50, shard: int = 0,
          nshards: int = 1, max_blocks: int | None = None, evaluate=None) -> dict:
    """Run (or resume) a sweep; returns the state.  max_blocks limits this call (for tests / time slicing)."""
    evaluate = evaluate or gpu_block_evaluator
    state = new_state(lo, hi, mode, block, near_bound, shard, nshards)
    if os.path.exists(state_path):
        with open(state_path) as f:
            old = json.load(f)
        if old.get("digest") != state["digest"] or _digest(old.get("config", {})) != state["digest"]:
            raise ValueError(f"{state_path}: checkpoint belongs to another sweep configuration "
                             "(or another partition / format version)")
        state = old
    todo = blocks_of(lo, hi, block, shard, nshards)
    if state["blocks"] != len(todo) or not 0 <= state["next_block"] <= len(todo):
        raise ValueError(f"{state_path}: checkpoint has {state['blocks']} blocks (next {state['next_block']}), "
                         f"this partition has {len(todo)}")
    done_now = 0
    while state["next_block"] < len(todo) and (max_blocks is None or done_now < max_blocks):
        a, b = todo[state["next_block"]]
        n, chk, hits, near, hw, hv = evaluate(a, b, mode, near_bound)
        state["primes"] += n
        state["checksum"] = str((int(state["checksum"]) + chk) & M64)
        state["hits"] = sorted(state["hits"] + [[str(p), f] for p, f in hits], key=lambda h: (int(h[0]), h[1]))
        state["near"] = sorted(state["near"] + [[str(p), t, s] for p, t, s in near], key=lambda x: (int(x[0]), x[1]))
        state["hist_w"] = [x + y for x, y in zip(state["hist_w"], hw)]
        state["hist_v"] = [x + y for x, y in zip(state["hist_v"], hv)]
        state["next_block"] += 1
        state["done"] = state["next_block"] == len(todo)
        _write(state_path, state)
        done_now += 1
    if not os.path.exists(state_path):
        _write(state_path, state)
    return state


def merge_states(states: list[dict]) -> dict:
    """Combine the per-shard states of one sweep into the unsharded state's outputs."""
    cfgs = {json.dumps({k: v for k, v in s["config"].items() if k not in ("shard",)}, sort_keys=True) for s in states}
    if len(cfgs) != 1:
        raise ValueError("states belong to different sweeps")
    nshards = states[0]["config"]["nshards"]
    if sorted(s["config"]["shard"] for s in states) != list(range(nshards)):
        raise ValueError(f"merge needs each shard 0..{nshards - 1} exactly once, got "
                         f"{sorted(s['config']['shard'] for s in states)}")
    cfg = dict(states[0]["config"], shard=0, nshards=1)
    out = dict(config=cfg, digest=_digest(cfg), done=all(s["done"] for s in states),
               primes=sum(s["primes"] for s in states),
               checksum=str(sum(int(s["checksum"]) for s in states) & M64),
               hits=sorted([h for s in states for h in s["hits"]], key=lambda h: (int(h[0]), h[1])),
               near=sorted([x for s in states for x in s["near"]], key=lambda x: (int(x[0]), x[1])),
               hist_w=[sum(v) for v in zip(*(s["hist_w"] for s in states))],
               hist_v=[sum(v) for v in zip(*(s["hist_v"] for s in states))])
    return out


def main(argv=None):
    """CLI: python -m paper_2101_11157_b200.sweep LO HI MODE STATE.json [--block B] [--shard S --nshards N]"""
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("lo", type=int)
    ap.add_argument("hi", type=int)
    ap.add_argument("mode", type=int)
    ap.add_argument("state")
    ap.add_argument("--block", type=int, default=1 << 22)
    ap.add_argument("--near-bound", type=int, default=50)
    ap.add_argument("--shard", type=int, default=0)
    ap.add_argument("--nshards", type=int, default=1)
    ap.add_argument("--max-blocks", type=int, default=None)
    a = ap.parse_args(argv)
    s = sweep(a.lo, a.hi, a.mode, a.block, a.state, a.near_bound, a.shard, a.nshards, a.max_blocks)
    print(json.dumps({k: s[k] for k in ("next_block", "blocks", "primes", "checksum", "hits", "near", "done")}))


if __name__ == "__main__":
    main()
