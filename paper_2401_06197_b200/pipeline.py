"""Host <-> device streaming for batches that live in host memory (plumbing only).

A batch whose inputs sit in pinned host memory is processed in image chunks over three
CUDA streams: the host->device copies of chunk c+1, the library calls of chunk c and the
device->host copies of chunk c-1 run concurrently (the copy engines of both directions
and the SMs overlap), ordered per chunk by CUDA events.  Across repeated runs a chunk's
inputs are not overwritten before the previous run's kernels of that chunk finished, and
its outputs not before the previous run's device->host copies of it finished.  No
compute happens here: `compute(c)` is the caller's sequence of library calls.
"""
from __future__ import annotations

from typing import Callable

import torch


class HostPipeline:
    def __init__(self, device: torch.device, chunks: int):
        self.device = device
        self.chunks = chunks
        self.s_in = torch.cuda.Stream(device=device)
        self.s_cmp = torch.cuda.Stream(device=device)
        self.s_out = torch.cuda.Stream(device=device)
        self._cmp_done = [None] * chunks
        self._out_done = [None] * chunks

    def run(self, h2d: Callable[[int], None], compute: Callable[[int], None],
            d2h: Callable[[int], None]):
        """Enqueue one pass over all chunks; returns the (start, end) CUDA events."""
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(self.s_in)
        self.s_cmp.wait_event(start)
        self.s_out.wait_event(start)
        for c in range(self.chunks):
            with torch.cuda.stream(self.s_in):
                if self._cmp_done[c] is not None:
                    self.s_in.wait_event(self._cmp_done[c])
                h2d(c)
                e_in = torch.cuda.Event()
                e_in.record(self.s_in)
            with torch.cuda.stream(self.s_cmp):
                self.s_cmp.wait_event(e_in)
                if self._out_done[c] is not None:
                    self.s_cmp.wait_event(self._out_done[c])
                compute(c)
                e_c = torch.cuda.Event()
                e_c.record(self.s_cmp)
                self._cmp_done[c] = e_c
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(e_c)
                d2h(c)
                e_o = torch.cuda.Event()
                e_o.record(self.s_out)
                self._out_done[c] = e_o
        self.s_out.wait_stream(self.s_in)
        self.s_out.wait_stream(self.s_cmp)
        end.record(self.s_out)
        return start, end
