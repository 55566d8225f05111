"""Gradient tape: record device ops on the forward pass, replay pullbacks.

The reference records pullback state in a persistent LIFO (``Tape``,
interp.py:38-61) filled by the augmented forward (``_Augmenter``,
reverse_ad.py:186-324) and drained by the pullback (reverse_ad.py:330-613);
the save set of every op is its rule's ``saves`` (rules.py:195-218).  Here
an entry holds the device buffers its adjoint needs (the same save set:
operands for matmul, the result for tanh/sigmoid) and a ``backward``
closure that enqueues the adjoint kernels on the current CUDA stream.

Replay is pure: the pullback reads the tape without consuming it, so it
can run several times against one forward (the DAN step pulls back two
seeds, nn_train.py:360-363), and a whole record/replay sequence can be
captured once into a CUDA graph (:meth:`Tape.capture`).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable


@dataclass
class TapeEntry:
    name: str
    saved: tuple
    backward: Callable  # backward(ctx) -> None, enqueues kernels
    on_done: Callable | None = None  # called after this entry's adjoint is enqueued


@dataclass
class Tape:
    entries: list = field(default_factory=list)

    def push(self, entry: TapeEntry) -> None:
        self.entries.append(entry)

    def __len__(self) -> int:
        return len(self.entries)

    def pullback(self, ctx=None) -> None:
        """Enqueue every adjoint in reverse recording order (LIFO)."""
        for e in reversed(self.entries):
            e.backward(ctx)
            if e.on_done is not None:
                e.on_done(e)

    def clear(self) -> None:
        self.entries.clear()

    @staticmethod
    def capture(fn: Callable, stream=None, warmup: int = 0):
        """Capture ``fn()`` (a full record + replay sequence) into a CUDA graph."""
        import torch

        s = stream or torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        # thread-local capture: NCCL's proxy threads (data-parallel steps) keep
        # making CUDA calls while this thread captures
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            fn()
        return g
