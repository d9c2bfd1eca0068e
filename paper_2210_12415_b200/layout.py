"""Layout primitives — the Python face of lf::LayoutPrimitive / PrimitiveSeq.

Mirrors proj/include/layoutforge/layout.hpp:19-59: six primitives
(split/reorder/fuse/unfold/pad/store_at) plus the inverses the reference
generates (fold/unpad/decouple_at). Dims are 0-based as in the reference's
C++ API. Shape derivation runs in the native library
(lfgpu_derive_layout), never in Python.
"""
from dataclasses import dataclass, field
from typing import List, Optional

from . import _abi

_KIND_NAMES = {
    _abi.SPLIT: "split",
    _abi.REORDER: "reorder",
    _abi.FUSE: "fuse",
    _abi.UNFOLD: "unfold",
    _abi.PAD: "pad",
    _abi.STORE_AT: "store_at",
    _abi.FOLD: "fold",
    _abi.UNPAD: "unpad",
    _abi.DECOUPLE_AT: "decouple_at",
}


@dataclass
class LayoutPrimitive:
    """lf::LayoutPrimitive (layout.hpp:33-52)."""

    kind: int
    dim: int = 0
    factors: List[int] = field(default_factory=list)
    perm: List[int] = field(default_factory=list)
    span: int = 0
    tile: int = 0
    stride: int = 0
    pad: int = 0
    orig_extent: int = 0
    target: Optional[str] = None  # store_at target tensor id

    # constructors named like the reference's static factories (layout.cpp:27-75)
    @staticmethod
    def split(dim, factors):
        return LayoutPrimitive(_abi.SPLIT, dim=dim, factors=list(factors))

    @staticmethod
    def reorder(perm):
        return LayoutPrimitive(_abi.REORDER, perm=list(perm))

    @staticmethod
    def fuse(first_dim, count):
        return LayoutPrimitive(_abi.FUSE, dim=first_dim, span=count)

    @staticmethod
    def unfold(dim, tile, stride):
        return LayoutPrimitive(_abi.UNFOLD, dim=dim, tile=tile, stride=stride)

    @staticmethod
    def padding(dim, size):
        return LayoutPrimitive(_abi.PAD, dim=dim, pad=size)

    @staticmethod
    def store_at(target, dim):
        return LayoutPrimitive(_abi.STORE_AT, dim=dim, target=target)

    @property
    def name(self):
        return _KIND_NAMES[self.kind]

    def fill(self, p, tensor_index=None):
        p.kind = self.kind
        p.dim = self.dim
        p.span = self.span
        p.nfactors = len(self.factors)
        for i, f in enumerate(self.factors):
            p.factors[i] = int(f)
        p.nperm = len(self.perm)
        for i, v in enumerate(self.perm):
            p.perm[i] = int(v)
        p.tile = self.tile
        p.stride = self.stride
        p.pad = self.pad
        p.orig_extent = self.orig_extent
        p.target = -1
        if self.target is not None:
            if tensor_index is None:
                raise ValueError("store_at needs graph context to resolve its target")
            p.target = tensor_index(self.target)

    @staticmethod
    def from_c(p, tensor_id=None):
        return LayoutPrimitive(
            kind=p.kind,
            dim=p.dim,
            factors=[p.factors[i] for i in range(p.nfactors)],
            perm=[p.perm[i] for i in range(p.nperm)],
            span=p.span,
            tile=p.tile,
            stride=p.stride,
            pad=p.pad,
            orig_extent=p.orig_extent,
            target=(tensor_id(p.target) if (p.target >= 0 and tensor_id) else None),
        )

    def __repr__(self):
        k = self.kind
        if k == _abi.SPLIT:
            return f"split({self.dim}, {self.factors})"
        if k == _abi.REORDER:
            return f"reorder({self.perm})"
        if k == _abi.FUSE:
            return f"fuse({self.dim}, {self.span})"
        if k == _abi.UNFOLD:
            return f"unfold({self.dim}, {self.tile}, {self.stride})"
        if k == _abi.PAD:
            return f"pad({self.dim}, {self.pad})"
        if k == _abi.STORE_AT:
            return f"store_at({self.target!r}, {self.dim})"
        return f"{self.name}(dim={self.dim})"


def split(dim, factors):
    return LayoutPrimitive.split(dim, factors)


def reorder(perm):
    return LayoutPrimitive.reorder(perm)


def fuse(first_dim, count):
    return LayoutPrimitive.fuse(first_dim, count)


def unfold(dim, tile, stride):
    return LayoutPrimitive.unfold(dim, tile, stride)


def padding(dim, size):
    return LayoutPrimitive.padding(dim, size)


def store_at(target, dim):
    return LayoutPrimitive.store_at(target, dim)
