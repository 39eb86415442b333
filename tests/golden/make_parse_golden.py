"""Generate tests/golden/parse_cases.json from the UNMODIFIED reference (oracle/_ref):
parse_edge_list (graph.cpp:136-172) on hand-written edge-list texts, including every
error branch, and on two larger random Gset texts.

    make -C oracle ref && python tests/golden/make_parse_golden.py

Each case records the text (or the seed that regenerates it), and either the resulting
CSR (n, m, sha256 of offsets / adjacency) or the reference's status and message.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

TEXTS = {
    "plain": "4 3\n1 2\n2 3\n3 4\n",
    "no_trailing_newline": "3 2\n1 2\n2 3",
    "comments_blank": "% a comment\n# another\n\n   \n3 3\n% mid comment\n1 2\n\n2 3\n  # indented\n1 3\n",
    "crlf": "3 2\r\n1 2\r\n2 3\r\n",
    "weights": "3 2\n1 2 1\n2 3 -1\n",
    "float_weights": "3 2\n1 2 0.5\n2 3 .25\n",
    "duplicates_both_orders": "4 5\n1 2\n2 1\n1 2\n3 4\n4 3\n",
    "tabs_and_spaces": "3\t2\n\t1 \t 2\n 2\t3   \n",
    "header_extra_tokens": "3 2 extra\n1 2\n2 3\n",
    "edge_extra_tokens": "3 2\n1 2 x y\n2 3\n",
    "isolated_nodes": "6 2\n1 2\n5 6\n",
    "no_edges": "5 0\n",
    "m_mismatch": "3 10\n1 2\n",
    "plus_sign": "3 2\n+1 2\n2 +3\n",
    "vtab_content": "3 2\n\v1 2\n2 3\n",
    "empty": "",
    "only_comments": "% nothing\n# here\n\n",
    "bad_header_one_token": "5\n1 2\n",
    "bad_header_zero_n": "0 0\n",
    "bad_header_negative_m": "3 -1\n1 2\n",
    "bad_header_text": "n m\n1 2\n",
    "bad_edge_one_token": "3 2\n1 2\n3\n",
    "bad_edge_text": "3 2\n1 2\nfoo bar\n",
    "bad_edge_float_id": "3 2\n1.5 2\n",
    "range_high": "3 2\n1 2\n2 4\n",
    "range_zero": "3 2\n0 2\n",
    "range_negative": "3 2\n1 -2\n",
    "self_loop": "3 2\n1 2\n3 3\n",
    "first_error_wins": "4 3\n1 2\n4 4\n1 9\n",
    "first_error_parse_before_loop": "4 3\nx y\n4 4\n",
    "overflow": "3 2\n1 99999999999999999999\n",
    "vtab_only_line": "3 1\n\v\n1 2\n",
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(text: bytes):
    try:
        rg = O.RefGraph.parse(text)
    except O.OracleError as e:
        return {"status": e.status, "message": str(e).split(": ", 1)[1]}
    off = np.zeros(rg.n + 1, dtype=np.int64)
    adj = np.zeros(max(2 * rg.m, 1), dtype=np.uint32)
    O.ref.ref_graph_csr(rg.h, O._ptr(off), O._ptr(adj))
    return {"status": 0, "n": rg.n, "m": rg.m, "off_sha": sha(off), "adj_sha": sha(adj[: 2 * rg.m])}


def random_gset(n, m, seed, weights):
    """A Gset-style text: header, m random (u, v) lines (1-based, no self-loops, repeats
    allowed), optional weight column, a comment line every 1000 edges."""
    rng = np.random.default_rng(seed)
    u = rng.integers(1, n + 1, m)
    v = rng.integers(1, n, m)
    v = np.where(v >= u, v + 1, v)
    lines = [f"{n} {m}"]
    for i in range(m):
        if i % 1000 == 0:
            lines.append(f"% block {i}")
        lines.append(f"{u[i]} {v[i]} 1" if weights else f"{u[i]} {v[i]}")
    return ("\n".join(lines) + "\n").encode()


def main():
    cases = {k: {"text": t, **outcome(t.encode())} for k, t in TEXTS.items()}
    rand = {}
    for name, (n, m, seed, w) in {"random_5k": (5000, 20000, 1, False), "random_w_20k": (20000, 60000, 2, True)}.items():
        rand[name] = {"lines": m, "seed": seed, "weights": w, **outcome(random_gset(n, m, seed, w))}
    with open(os.path.join(OUT, "parse_cases.json"), "w") as f:
        json.dump({"cases": cases, "random": rand}, f, indent=1)
    print(f"{len(cases)} texts, {len(rand)} random Gset files")


if __name__ == "__main__":
    main()
