"""The SPEC's executor plugin point, B200-native.

The reference's ``LocalExecutor`` (executor.py:52-94) runs SPMD workers in
synchronous supersteps and routes messages between them.  On B200 the
workers of one TSQR are the CTAs of the leaf kernel and the combine events of
the tree kernels; the cross-GPU level is one process per GPU exchanging R
factors over NCCL (``paper_0809_2407_b200.dist``).  ``DeviceExecutor`` carries
the device and stream the kernels run on plus a ``CommRecorder`` per logical
worker, so the reference's census (messages / words per tree level) stays
observable.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .counters import CommRecorder


class ExecutorError(RuntimeError):
    """Device or communication failure (executor.py:48-49)."""


@dataclass
class DeviceExecutor:
    """One CUDA device (and stream) that runs the TSQR/CAQR kernels.

    ``record=True`` fills per-leaf CommRecorders with the packed-R messages the
    tree implies (n(n+1)/2 words per combine).
    """

    device: int = 0
    stream: object = None
    record: bool = False
    recorders: list = field(default_factory=list)

    def torch_device(self):
        import torch

        return torch.device("cuda", self.device)

    def cuda_stream(self):
        import torch

        st = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
        return st

    def stream_handle(self) -> int:
        return int(self.cuda_stream().cuda_stream)

    def census(self, tree, n: int) -> None:
        if not self.record:
            return
        self.recorders = [CommRecorder() for _ in range(tree.P)]
        words = n * (n + 1) // 2
        for ev in tree.schedule():
            recv = ev.receiver
            for p in ev.participants:
                if p == recv:
                    continue
                self.recorders[p].record_send(words)
                self.recorders[recv].record_recv(words, stage=(ev.level, "R"))


def LocalExecutor(threads: int = 1):  # noqa: N802 - reference name
    """Reference-compatible constructor: the GPU executor on the current device."""
    if threads < 1:
        raise ValueError("threads must be >= 1")
    return DeviceExecutor()
