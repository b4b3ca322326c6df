"""HBM expert slot pool: one [n_slots, numel] tensor holding experts as flat
vectors [W_in | W_out] — the layout the grouped-GEMM tensor maps address
with the slot as the outer coordinate, so resident experts are never copied
to be computed on, merged experts are written straight into free slots and
singleton groups alias their principal's slot."""

from __future__ import annotations

import torch


class ExpertPool:
    def __init__(self, n_slots: int, numel: int, dtype=torch.bfloat16, device="cuda"):
        if n_slots < 1 or numel < 1:
            raise ValueError("pool needs at least one slot of at least one element")
        pad = (-numel) % 64  # keep every slot 128-byte aligned
        self.numel = int(numel)
        self.stride = int(numel + pad)
        self.data = torch.empty((n_slots, self.stride), dtype=dtype, device=device)
        self._free = list(range(n_slots - 1, -1, -1))

    @property
    def n_slots(self) -> int:
        return self.data.shape[0]

    @property
    def dtype(self):
        return self.data.dtype

    @property
    def slot_bytes(self) -> int:
        return self.numel * self.data.element_size()

    def alloc(self, exclude=()) -> int:
        """A free slot, never one of `exclude` (e.g. slots holding experts
        that were written through `data` without alloc(): they are reserved
        on the way, so later allocations skip them too)."""
        ex = set(exclude)
        for s in [s for s in self._free if s in ex]:
            self._free.remove(s)
        if not self._free:
            raise RuntimeError("expert pool is full")
        return self._free.pop()

    def reserve(self, slot: int) -> None:
        """Mark a slot filled through `data` as in use."""
        if slot in self._free:
            self._free.remove(slot)

    def release(self, slot: int) -> None:
        if not 0 <= slot < self.n_slots or slot in self._free:
            raise ValueError(f"bad slot {slot}")
        self._free.append(slot)

    def free_slots(self) -> int:
        return len(self._free)

    def view(self, slot: int) -> torch.Tensor:
        return self.data[slot, : self.numel]

    def slot_of(self, t: torch.Tensor):
        """Slot index if `t` is exactly one slot view of this pool, else None."""
        if not isinstance(t, torch.Tensor) or t.numel() != self.numel:
            return None
        off = t.data_ptr() - self.data.data_ptr()
        row = self.stride * self.data.element_size()
        if off < 0 or off % row or off // row >= self.n_slots:
            return None
        return off // row
