"""Stable sub-seed derivation (mirror of ``coesim.seeding``, seeding.py:15-19).

A child seed is the first 8 bytes (big endian) of SHA-256 over
``"<seed>/<label>/<label>..."``; it is stable across processes, unlike ``hash``.
"""

from __future__ import annotations

import hashlib


def subseed(seed: int, *labels: object) -> int:
    path = "/".join([str(int(seed)), *(str(label) for label in labels)])
    return int.from_bytes(hashlib.sha256(path.encode("utf-8")).digest()[:8], "big")
