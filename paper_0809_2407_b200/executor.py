"""The SPEC's executor plugin point, B200-native.

The reference's ``LocalExecutor`` (executor.py:52-94) runs SPMD worker
programs in synchronous supersteps and routes messages between them.  On B200
the workers of one TSQR are the CTAs of the leaf kernel and the combine
events of the tree kernels; the cross-GPU level is one process per GPU
exchanging R factors over NCCL (``paper_0809_2407_b200.dist``).

Two things live here:

* ``DeviceExecutor``: the GPU group the TSQR / CAQR kernels run on (device,
  stream) plus a ``CommRecorder`` per logical worker, so the reference's
  census (messages / words per tree level) stays observable.
* ``LocalExecutor``: the reference's host-side SPMD runner, kept API-compatible
  for callers that drive their own worker programs (``run(program)`` returns
  ``(results, recorders)``; ``Message``, ``payload_words``).  It is control
  plane, not the hot path: passing it to ``tsqr_parallel`` runs the GPU path
  on its device like a ``DeviceExecutor``.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from .counters import CommRecorder


class ExecutorError(RuntimeError):
    """Device, communication or worker failure (executor.py:48-49)."""


def payload_words(payload) -> int:
    """Float words a message carries (executor.py:20-33): arrays count their
    elements, scalars one, containers the sum of their items."""
    if payload is None:
        return 0
    if isinstance(payload, np.ndarray):
        return int(payload.size)
    numel = getattr(payload, "numel", None)  # torch tensors
    if callable(numel) and not isinstance(payload, (int, float)):
        return int(numel())
    if isinstance(payload, (bool, int, float, np.integer, np.floating)):
        return 1
    if isinstance(payload, dict):
        return sum(payload_words(v) for v in payload.values())
    if isinstance(payload, (list, tuple)):
        return sum(payload_words(v) for v in payload)
    return 0


@dataclass
class Message:
    """A routed message (executor.py:36-45); ``words`` defaults to the payload's."""

    src: int
    dst: int
    tag: str
    payload: object
    words: int = field(default=-1)

    def __post_init__(self):
        if self.words < 0:
            self.words = payload_words(self.payload)


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


class LocalExecutor(DeviceExecutor):
    """Reference-compatible SPMD runner (executor.py:52-94) that is also a GPU executor.

    ``run(program)``: ``program`` has ``n_workers``, ``n_steps``, ``setup(w)``,
    ``step(w, state, step, inbox) -> messages`` and ``finish(w, state)``.  Each
    superstep runs every worker (on a thread pool when ``threads > 1``), then
    delivers the messages; inboxes are ordered by (src, tag) so the result
    does not depend on the thread count.  A worker exception, a forged
    sender or an unknown destination raise ``ExecutorError``.
    """

    def __init__(self, threads: int = 1, device: int = 0, stream=None, record: bool = False):
        if threads < 1:
            raise ValueError("threads must be >= 1")
        super().__init__(device=device, stream=stream, record=record)
        self.threads = threads

    def run(self, program):
        P = program.n_workers
        states = [program.setup(w) for w in range(P)]
        recs = [CommRecorder() for _ in range(P)]
        inbox = [[] for _ in range(P)]

        def one(w, step):
            try:
                return program.step(w, states[w], step, inbox[w])
            except Exception as exc:  # noqa: BLE001 - surfaced as the executor's error
                raise ExecutorError(f"worker {w} failed at step {step}: {exc}") from exc

        for step in range(program.n_steps):
            if self.threads > 1 and P > 1:
                with ThreadPoolExecutor(max_workers=min(self.threads, P)) as pool:
                    sent = list(pool.map(lambda w: one(w, step), range(P)))
            else:
                sent = [one(w, step) for w in range(P)]
            nxt = [[] for _ in range(P)]
            for w, msgs in enumerate(sent):
                for msg in msgs or ():
                    if msg.src != w:
                        raise ExecutorError(f"worker {w} sent a message as worker {msg.src}")
                    if not 0 <= msg.dst < P:
                        raise ExecutorError(f"message to unknown worker {msg.dst}")
                    recs[w].record_send(msg.words)
                    nxt[msg.dst].append(msg)
            for dst in range(P):
                nxt[dst].sort(key=lambda m: (m.src, m.tag))
                for msg in nxt[dst]:
                    recs[dst].record_recv(msg.words, stage=(step, msg.tag))
            inbox = nxt
        return [program.finish(w, states[w]) for w in range(P)], recs
