"""Generate tests/golden/*.npz from the REAL reference (oracle/_ref, compiled
from /root/reference/proj/src by oracle/Makefile). Run here, where
/root/reference exists; the committed fixtures travel to the GPU box.

    make -C oracle ref && python tests/golden/make_golden.py

Each case records seeded inputs and the reference's outputs:
select() plans, logits() bit patterns and greedy_step() ids. The reference's
golden plan file is copied verbatim as the wire-format fixture.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import ref_lib, words_from_ids  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def splitmix(seed, n):
    g = np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + np.arange(1, n + 1, dtype=np.uint64) * g
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def bf16(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return ((((u + np.uint32(0x7FFF) + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32)
            .view(np.float32))


# (name, V, d, n_static, L, B, dtype_bytes, bf16, seed)
CASES = [
    ("tiny_f32", 200, 7, 11, 9, 3, 4, False, 1),
    ("odd_f32", 1000, 33, 40, 50, 4, 4, False, 2),
    ("f16_rt", 777, 64, 30, 40, 3, 2, False, 3),
    ("bf16_d96", 4096, 96, 128, 96, 4, 4, True, 4),
    ("f32_d256", 5000, 256, 200, 120, 2, 4, False, 5),
    ("empty_static", 300, 16, 0, 20, 2, 4, False, 6),
    ("empty_prompt", 300, 16, 25, 0, 2, 4, False, 7),
]


def main():
    ref = ref_lib()
    for name, V, d, ns, L, B, db, use_bf16, seed in CASES:
        W = ref.head_random(V, d, 0x5EED + seed, db)
        if use_bf16:
            W = bf16(W)
        st = np.unique((splitmix(0x57A7 + seed, ns * 4) % np.uint64(V)).astype(np.uint32))[:ns]
        words = words_from_ids(st, V)
        prompts = [(splitmix(0x9A0 + 97 * seed + b, L) % np.uint64(V)).astype(np.uint32)
                   for b in range(B)]
        # repeated ids inside the prompt exercise the dedup path
        for p in prompts:
            if len(p) > 4:
                p[len(p) // 2] = p[0]
        hid = ref.head_random(B, d, 0x41DD + seed, 4)
        if use_bf16:
            hid = bf16(hid)
        plans, ns_, nd_, logit_bits, greedy = [], [], [], [], []
        for b in range(B):
            pl = ref.select(prompts[b], words, V, V)
            plans.append(pl.active_ids)
            ns_.append(pl.n_static)
            nd_.append(pl.n_dynamic)
            sub = ref.gather(W, pl.active_ids)
            logit_bits.append(ref.logits(sub, hid[b]).view(np.uint32))
            greedy.append(ref.greedy_step(sub, hid[b], pl.active_ids) if len(pl.active_ids) else
                          np.uint32(0xFFFFFFFF))
        off = np.zeros(B + 1, np.int64)
        off[1:] = np.cumsum([len(p) for p in plans])
        poff = np.zeros(B + 1, np.int64)
        poff[1:] = np.cumsum([len(p) for p in prompts])
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"), V=V, d=d, dtype_bytes=db, bf16=use_bf16,
            W_seed=0x5EED + seed, H_seed=0x41DD + seed,
            W_sha256=hashlib.sha256(W.view(np.uint32).tobytes()).hexdigest(),
            hidden_bits=hid.view(np.uint32), static_ids=st,
            prompts=np.concatenate(prompts) if L else np.zeros(0, np.uint32), prompt_off=poff,
            plan_ids=np.concatenate(plans), plan_off=off, n_static=np.array(ns_),
            n_dynamic=np.array(nd_), logit_bits=np.concatenate(logit_bits),
            greedy=np.array(greedy, np.uint32))
        print("wrote", name)


def copy_plan_fixture():
    """The reference's own golden plan file (fixtures/golden/plan_aca.json,
    the output of its save_json: nlohmann dump(2) + newline) pins the plan
    wire format (tests/test_plan_json.py)."""
    src = "/root/reference/proj/tests/fixtures/golden/plan_aca.json"
    with open(src, "rb") as f, open(os.path.join(OUT, "plan_aca.json"), "wb") as g:
        g.write(f.read())


if __name__ == "__main__":
    main()
    copy_plan_fixture()
