"""Multi-GPU fit over the shard ABI (include/ig_b200.h).

One process per GPU.  Training rows are replicated: every rank encodes the same
columns.  Per class, each rank deduplicates the pairs of its round-robin share
of the pair-tile triangle, routes the distinct candidates to their owner rank
(content fingerprint mod world) as 8-byte (u, v) row-pair records, and the
records are exchanged with one all-to-all (NCCL over NVLink/NVSwitch through
torch.distributed).  Owners deduplicate exactly across ranks and run support /
score / coverage on what they own; the matcher's per-rank partial A/N are
summed with one all-reduce.  No other data moves.

The same shard ABI also runs as an in-process emulation of `world` ranks on one
device (`fit_emulated`, used by the single-GPU tests), where the "all-to-all"
is a concatenation of the per-rank send slices.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

from .api import Context, Encoding, IGArithmeticError, KernelConfig, Model, lib

INT64_MAX = (1 << 63) - 1


def _torch_stream(ctx: Context):
    """The library runs on torch's current stream while it reads or writes
    tensors torch produced or consumes (all-to-all receive buffers, evidence
    outputs): a context's own stream is non-blocking and not ordered with it."""
    import torch
    if not torch.cuda.is_available() or not hasattr(ctx, "on_stream"):
        import contextlib
        return contextlib.nullcontext()
    return ctx.on_stream(torch.cuda.current_stream())


class _CudaArray:
    """Zero-copy view of a library-owned device buffer (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<i8"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr or 0, False),
                                         "version": 3, "strides": None}


class _ShardModel(Model):
    """The owned dictionaries of a shard (memory owned by the shard, which this
    view keeps alive)."""

    def __init__(self, ctx: Context, handle, owner: "Shard"):
        super().__init__(ctx, handle)
        self._owner = owner

    def __del__(self):
        self.handle = None


class Shard:
    def __init__(self, ctx: Context, enc: Encoding, rank: int, world: int, config: Optional[KernelConfig] = None):
        cfg = (config or KernelConfig()).c()
        h = C.c_void_p()
        ctx.check(lib.ig_shard_create(ctx.handle, enc.handle, rank, world, C.byref(cfg), C.byref(h)))
        self.ctx, self.enc, self.rank, self.world, self.handle = ctx, enc, rank, world, h

    def enumerate(self, cls: int):
        """-> (counts[world] records per destination, int64 tensor view of the send buffer,
        records grouped by destination; valid until the next enumerate of this class)."""
        import torch
        counts = (C.c_uint64 * self.world)()
        ptr = C.c_void_p()
        self.ctx.check(lib.ig_shard_enumerate(self.ctx.handle, self.handle, cls, counts, C.byref(ptr)))
        counts = [int(x) for x in counts]
        n = sum(counts)
        send = torch.as_tensor(_CudaArray(int(ptr.value or 0), n), device="cuda") if n else \
            torch.empty(0, dtype=torch.int64, device="cuda")
        return counts, send

    def receive(self, cls: int, recv, n_records: int) -> None:
        """recv: int64 device tensor holding n_records (u, v) records."""
        self.ctx.check(lib.ig_shard_receive(self.ctx.handle, self.handle, cls,
                                            C.c_void_p(recv.data_ptr() if n_records else None), n_records))

    def finish(self) -> tuple[int, int]:
        tot = (C.c_uint64 * 2)()
        self.ctx.check(lib.ig_shard_finish(self.ctx.handle, self.handle, tot))
        return int(tot[0]), int(tot[1])

    @property
    def model(self) -> Model:
        return _ShardModel(self.ctx, lib.ig_shard_model(self.handle), self)

    def partial_evidence(self, tenc: Encoding):
        """A/N of the owned dictionaries only (int64 device tensors)."""
        import torch
        n = tenc.rows(2)
        dA = torch.zeros(n, dtype=torch.int64, device="cuda")
        dN = torch.zeros(n, dtype=torch.int64, device="cuda")
        if n:
            # the encoding's background index of the test rows (ig_encode_rows) is reused;
            # torch's stream: dA / dN were zeroed there and are all-reduced there
            with _torch_stream(self.ctx):
                self.model.evidence_encoded_device(tenc, dA.data_ptr(), dN.data_ptr())
        return dA, dN

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:  # lib is None at interpreter teardown
            lib.ig_shard_free(self.handle)
            self.handle = None


class TorchExchange:
    """all-to-all / all-gather / all-reduce over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())

    def all_to_all(self, send, counts: list[int]):
        """int64 records grouped by destination; returns (recv tensor, n records)."""
        recv, n, work = self.all_to_all_start(send, counts)
        work.wait()
        return recv, n

    def all_to_all_start(self, send, counts: list[int]):
        """The same, asynchronously: the counts are exchanged at once (they size
        the receive buffer), the records in flight when this returns; call
        .wait() on the returned work before reading recv (on NCCL it orders the
        current stream after the transfer without blocking the host)."""
        import torch
        world = len(counts)
        dev = self.device
        cin = torch.tensor(counts, dtype=torch.int64, device=dev)
        cout = torch.empty(world, dtype=torch.int64, device=dev)
        self.dist.all_to_all_single(cout, cin, group=self.group)
        rc = cout.tolist()
        recv = torch.empty(max(sum(rc), 1), dtype=torch.int64, device=dev)
        work = self.dist.all_to_all_single(recv[:sum(rc)], send, output_split_sizes=rc, input_split_sizes=counts,
                                           group=self.group, async_op=True)
        return recv, sum(rc), work

    def all_gather_ints(self, vals: list[int]) -> list[list[int]]:
        import torch
        dev = self.device
        t = torch.tensor([v & ((1 << 63) - 1) for v in vals] + [v >> 63 for v in vals], dtype=torch.int64, device=dev)
        out = [torch.empty_like(t) for _ in range(self.dist.get_world_size(self.group))]
        self.dist.all_gather(out, t, group=self.group)
        n = len(vals)
        return [[int(x[i]) | (int(x[n + i]) << 63) for i in range(n)] for x in (o.tolist() for o in out)]

    def all_reduce_sum_(self, tensor) -> None:
        self.dist.all_reduce(tensor, group=self.group)


def _check_totals(per_rank: list[list[int]]) -> None:
    for c in range(2):
        if sum(r[c] for r in per_rank) > INT64_MAX:
            raise IGArithmeticError("total score overflows int64")


@dataclass
class ShardedResult:
    shard: Shard
    model: Model


def fit_distributed(ctx: Context, enc: Encoding, rank: int, world: int, exchange: TorchExchange,
                    config: Optional[KernelConfig] = None, shard_factory=None) -> ShardedResult:
    """This rank's part of the sharded fit (call on every rank).  shard_factory
    lets the CPU tests drive the same orchestration with an oracle-backed shard."""
    with _torch_stream(ctx):
        sh = (shard_factory or Shard)(ctx, enc, rank, world, config)
        # class 0's records travel while class 1 enumerates, class 1's while
        # class 0's owners deduplicate (a class's send buffer stays valid until
        # that class is enumerated again)
        c0, s0 = sh.enumerate(0)
        r0, n0, w0 = exchange.all_to_all_start(s0, c0)
        c1, s1 = sh.enumerate(1)
        r1, n1, w1 = exchange.all_to_all_start(s1, c1)
        w0.wait()
        sh.receive(0, r0, n0)
        w1.wait()
        sh.receive(1, r1, n1)
        totals = sh.finish()
    _check_totals(exchange.all_gather_ints(list(totals)))
    return ShardedResult(sh, sh.model)


def evidence_distributed(res: ShardedResult, tenc, exchange: TorchExchange):
    """Partial A/N of this rank's dictionaries summed over ranks (exact: totals checked)."""
    dA, dN = res.shard.partial_evidence(tenc)
    exchange.all_reduce_sum_(dA)
    exchange.all_reduce_sum_(dN)
    return dA, dN


def fit_emulated(ctx: Context, enc: Encoding, world: int, config: Optional[KernelConfig] = None) -> list[Shard]:
    """Run `world` ranks' shards one after another on one device; the all-to-all
    is the concatenation of every rank's send slice for each destination."""
    import torch
    with _torch_stream(ctx):
        shards = [Shard(ctx, enc, r, world, config) for r in range(world)]
        for cls in range(2):
            outs = [(counts, send.clone()) for counts, send in (sh.enumerate(cls) for sh in shards)]
            for r, sh in enumerate(shards):
                parts = [t[sum(counts[:r]):sum(counts[:r]) + counts[r]] for counts, t in outs]
                recv = torch.cat(parts) if parts else torch.empty(0, dtype=torch.int64, device="cuda")
                sh.receive(cls, recv, int(recv.numel()))
        _check_totals([list(sh.finish()) for sh in shards])
    return shards
