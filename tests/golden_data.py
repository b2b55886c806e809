"""Loaders for the committed golden vectors (tests/golden/*.npz).

The vectors were produced by running the reference implementation
(/root/reference/pkg/src/exsum) -- see tests/golden/make_golden.py.
"""

from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

MONO_DTYPE = {
    "add-i64": np.int64,
    "max-i64": np.int64,
    "add-f64": np.float64,
    "add-f32": np.float32,
}
MONO_OP = {"add-i64": "add", "max-i64": "max", "add-f64": "add", "add-f32": "add"}


@functools.lru_cache(maxsize=None)
def load(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def small_cases():
    """Yield (index, ext, box, inputs-by-monoid, outputs dict) for small.npz."""
    z = load("small")
    meta = json.loads(bytes(z["meta"]).decode())
    for ci, m in enumerate(meta):
        ext, box = tuple(m["ext"]), tuple(m["box"])
        ins = {
            "add-i64": z[f"{ci}/int"],
            "max-i64": z[f"{ci}/int"],
            "add-f64": z[f"{ci}/f64"],
            "add-f32": z[f"{ci}/f64"].astype(np.float32),
        }
        outs = {k.split("/", 1)[1]: v for k, v in z.items() if k.startswith(f"{ci}/")}
        yield ci, ext, box, ins, outs


def medium_cases():
    """Yield dicts with key/name/mono/route/box/ext plus 'in' and 'out' arrays."""
    z = load("medium")
    meta = json.loads(bytes(z["meta"]).decode())
    for m in meta:
        m = dict(m)
        m["in"] = z[f"{m['name']}/in/{m['mono']}"]
        m["out"] = z[m["key"]]
        yield m


def mono_op(mono: str) -> str:
    """Oracle / device operator string for a monoid name ("mod-add:<m>" passes through)."""
    return mono if mono.startswith("mod-add:") else MONO_OP[mono]


def ext_cases():
    """Yield dicts (key, mono, route, box, ext, 'in', 'out') for ext.npz: the
    sat/satc and mod-add vectors."""
    z = load("ext")
    meta = json.loads(bytes(z["meta"]).decode())
    for m in meta:
        m = dict(m)
        m["out"] = z[m["key"]]
        m["in"] = z[m["in"]]
        yield m


def corner_cases():
    """Yield dicts (tag, mono, box, ext, 'in', 'out') for corners.npz
    (corners_excluded / corners_spine_excluded, which agree bit for bit)."""
    z = load("corners")
    meta = json.loads(bytes(z["meta"]).decode())
    for m in meta:
        m = dict(m)
        m["in"] = z[m["tag"] + "/in"]
        m["out"] = z[m["tag"] + "/out"]
        yield m
