"""Block-vector container (reference: pintlab/linalg.py:58-120).

The interface states lambda_0..lambda_p are stored as one (P+1) x dim
row-major, slice-major array — here a device tensor in HBM. ``.data`` keeps
the reference's read contract (a numpy array) through a host copy made on
demand; that copy is READ-ONLY (writing into it raises instead of being
silently lost — the device tensor is the storage), and it is refreshed
whenever the tensor has been modified in place since. ``.tensor`` is the
device view used by the hot path; mutate state through it.
"""
from __future__ import annotations

import numpy as np
import torch

from .errors import DimensionError


class BlockVector:
    __slots__ = ("tensor", "_host", "_host_version")

    def __init__(self, data, check_finite: bool = True):
        if isinstance(data, torch.Tensor):
            t = data
        else:
            a = np.asarray(data, dtype=float)
            t = torch.from_numpy(np.ascontiguousarray(a))
        if t.dim() != 2:
            raise DimensionError(f"block vector needs a (n_blocks, dim) array, got ndim={t.dim()}")
        if check_finite and not bool(torch.isfinite(t).all()):
            raise ValueError("block entries must be finite")
        self.tensor = t
        self._host = None
        self._host_version = -1

    @classmethod
    def from_blocks(cls, blocks) -> "BlockVector":
        return cls(np.stack([np.asarray(b, dtype=float) for b in blocks]))

    @classmethod
    def from_flat(cls, flat, n_blocks: int) -> "BlockVector":
        """Reshape a flat vector into ``n_blocks`` equal blocks (linalg.py:96)."""
        a = np.asarray(flat, dtype=float).reshape(-1)
        if n_blocks <= 0 or a.size % n_blocks:
            raise DimensionError(f"cannot split {a.size} entries into {n_blocks} blocks")
        return cls(a.reshape(n_blocks, -1))

    @property
    def data(self) -> np.ndarray:
        """Read-only host copy (numpy) of the blocks (the reference's
        ``BlockVector.data`` for reading); refreshed after in-place changes of
        the device tensor."""
        ver = self.tensor._version
        if self._host is None or self._host_version != ver:
            h = self.tensor.detach().to("cpu").numpy()
            h.flags.writeable = False
            self._host = h
            self._host_version = ver
        return self._host

    @property
    def n_blocks(self) -> int:
        return int(self.tensor.shape[0])

    @property
    def block_dim(self) -> int:
        return int(self.tensor.shape[1])

    @property
    def flat(self) -> np.ndarray:
        return self.data.reshape(-1)

    def __getitem__(self, i: int) -> np.ndarray:
        return self.data[i]

    def __sub__(self, other: "BlockVector") -> "BlockVector":
        if tuple(self.tensor.shape) != tuple(other.tensor.shape):
            raise DimensionError("block vectors differ in shape")
        return BlockVector(self.tensor - other.tensor.to(self.tensor.device), check_finite=False)

    def copy(self) -> "BlockVector":
        return BlockVector(self.tensor.clone(), check_finite=False)

    def max_abs(self) -> float:
        """Unweighted infinity norm over every entry of every block."""
        if self.tensor.numel() == 0:
            return 0.0
        return float(self.tensor.abs().max())

    def __repr__(self) -> str:  # pragma: no cover
        return f"BlockVector(n_blocks={self.n_blocks}, dim={self.block_dim}, device={self.tensor.device})"
