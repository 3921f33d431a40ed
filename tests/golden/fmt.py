"""Shared (de)serialisation of golden cases (plain JSON, gzip-compressed).

Intervals are stored as exact rationals [num, den]; floats as `float.hex()` so
every golden comparison is bit-exact.
"""

from __future__ import annotations

import gzip
import json
from fractions import Fraction
from pathlib import Path

HERE = Path(__file__).resolve().parent


def enc_inv(model_shards, cache_shards):
    m = [[int(l), lo.numerator, lo.denominator, hi.numerator, hi.denominator]
         for l, lo, hi in model_shards]
    c = [[rid, int(l), lo.numerator, lo.denominator, hi.numerator, hi.denominator, int(t)]
         for rid, l, lo, hi, t in cache_shards]
    return {"m": m, "c": c}


def dec_inv(doc):
    m = tuple((l, Fraction(a, b), Fraction(c, d)) for l, a, b, c, d in doc["m"])
    c = tuple((rid, l, Fraction(a, b), Fraction(c2, d), t) for rid, l, a, b, c2, d, t in doc["c"])
    return m, c


def hx(x: float) -> str:
    return float(x).hex()


def unhx(s: str) -> float:
    return float.fromhex(s)


def save(name: str, doc):
    path = HERE / f"{name}.json.gz"
    with gzip.open(path, "wt", encoding="utf-8") as f:
        json.dump(doc, f, separators=(",", ":"), sort_keys=True)
    return path


def load(name: str):
    with gzip.open(HERE / f"{name}.json.gz", "rt", encoding="utf-8") as f:
        return json.load(f)
