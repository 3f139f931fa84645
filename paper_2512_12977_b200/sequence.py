"""Token layout: text / image segments (reference: model.py:35-106)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exceptions import InputError


@dataclass(frozen=True)
class Segment:
    kind: str  # "text" | "image"
    image_index: int | None
    start: int
    length: int


@dataclass
class TokenSequence:
    """Token ids (image positions carry -1) plus the segment map."""

    ids: list[int]
    segments: list[Segment]

    def __len__(self) -> int:
        return len(self.ids)

    @property
    def image_segments(self) -> list[Segment]:
        return [s for s in self.segments if s.kind == "image"]

    def validate(self, tokens_per_image: int | None = None) -> None:
        at, img = 0, 0
        for seg in self.segments:
            if seg.start != at:
                raise InputError(f"segments do not partition the sequence at {at}")
            if seg.length <= 0:
                raise InputError("empty segment")
            if seg.kind == "image":
                if seg.image_index != img:
                    raise InputError("image segments must be numbered in order")
                if tokens_per_image is not None and seg.length != tokens_per_image:
                    raise InputError(f"image segment length {seg.length} != tokens_per_image {tokens_per_image}")
                img += 1
            elif seg.kind != "text":
                raise InputError(f"unknown segment kind {seg.kind!r}")
            at += seg.length
        if at != len(self.ids):
            raise InputError("segments do not cover the id list")

    def image_mask(self) -> np.ndarray:
        m = np.zeros(len(self.ids), dtype=bool)
        for s in self.image_segments:
            m[s.start:s.start + s.length] = True
        return m


def make_sequence(prefix, num_images: int, tokens_per_image: int, suffix=()) -> TokenSequence:
    """text prefix, `num_images` image spans of `tokens_per_image`, text suffix."""
    ids: list[int] = [int(t) for t in prefix]
    segs: list[Segment] = [Segment("text", None, 0, len(ids))] if ids else []
    for m in range(num_images):
        segs.append(Segment("image", m, len(ids), tokens_per_image))
        ids.extend([-1] * tokens_per_image)
    if len(suffix):
        segs.append(Segment("text", None, len(ids), len(suffix)))
        ids.extend(int(t) for t in suffix)
    seq = TokenSequence(ids, segs)
    seq.validate(tokens_per_image if num_images else None)
    return seq
