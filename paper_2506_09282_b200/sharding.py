"""Multi-GPU partitioning of batched HDC inference (one process per GPU).

Two partitions, following the paper's two Stage II variants:

* N-shard (ScalableHD-L, Alg. 4, text P:410): rows of X are split
  across ranks; B and C are replicated; each rank runs the whole fused path on
  its rows; the only collective is an all-gather of the int32 labels (and,
  optionally, scores).  Rows are independent and the tensor-core kernels sum each
  row's Stage II tiles exactly (int64), so labels and scores equal the single-GPU ones
  bit for bit (tests/test_gpu_nshard.py); the fp32 FFMA kernels up to fp32 order.

* D-shard (ScalableHD-S, Alg. 3, text P:355): rank r holds the column
  slice D_r of B and C; it computes the partial scores S_r = HardSign(X B_r) C_r^T
  (hdc_model_partial_scores), the ranks sum them with one all-reduce of N x K
  fp32 (Alg. 3 `S += S_local`) and take the lowest-index argmax.

* D-shard with the reduction in the kernel (``DShardExchange``, SURVEY §8 f2 over peer
  memory): the small-batch kernel's last CTA stores S_r into every rank's exchange
  buffer (torch symmetric memory, peer-mapped), signals, waits for all ranks and sums
  the partials in rank order -- one launch, no NCCL call, identical results on all
  ranks.

torch.distributed (NCCL on GPUs) is plumbing only.  The per-rank compute is
delegated to an object with the ``Model`` interface (``infer`` /
``partial_scores``), normally ``paper_2506_09282_b200.Model``.
"""
import torch
import torch.distributed as dist


def shard_bounds(total, world, rank, align=1):
    """[lo, hi) of `rank`'s contiguous share of `total` items, boundaries rounded
    to multiples of `align` (the last rank takes the remainder)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    units = (total + align - 1) // align
    lo = (units * rank // world) * align
    hi = (units * (rank + 1) // world) * align
    return min(lo, total), min(hi, total)


def d_shard_slices(D, world, align=4):
    """Column slices of the D-shard: widths multiples of `align` (16-byte rows
    for fp32) except possibly the last."""
    return [shard_bounds(D, world, r, align) for r in range(world)]


def _gather_rows(local, counts, group=None):
    """All-gather variable-length row blocks (padded to the max count)."""
    world = dist.get_world_size(group)
    m = max(counts)
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


def shard_n_infer(model, X_local, N_total, return_scores=False, group=None):
    """N-shard inference: this rank holds rows [lo, hi) of X (its shard_bounds);
    returns all N_total labels (and scores) on every rank."""
    world = dist.get_world_size(group)
    counts = [hi - lo for lo, hi in (shard_bounds(N_total, world, r) for r in range(world))]
    rank = dist.get_rank(group)
    if X_local.shape[0] != counts[rank]:
        raise ValueError("X_local has %d rows, shard %d expects %d" % (X_local.shape[0], rank, counts[rank]))
    y, S = model.infer(X_local, return_scores=return_scores)
    labels = _gather_rows(y, counts, group)
    scores = _gather_rows(S, counts, group) if return_scores else None
    return labels, scores


class NShardGather:
    """The N-shard's one collective as the benchmark times it: every rank's int32 labels
    into one preallocated buffer with a single ``all_gather_into_tensor`` (shards padded to
    the largest, ScalableHD-L's "write y^(t') to global", Alg. 4).  ``labels`` is this
    rank's label buffer (write the shard's labels into it), ``gather()`` enqueues the
    collective and ``result()`` returns the N_total labels in row order."""

    def __init__(self, N_total, group=None, device=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.N = N_total
        self.bounds = [shard_bounds(N_total, self.world, r) for r in range(self.world)]
        self.counts = [hi - lo for lo, hi in self.bounds]
        self.pad = max(self.counts) if self.counts else 0
        self.buf = torch.zeros(self.pad, dtype=torch.int32, device=device)
        self.labels = self.buf[: self.counts[self.rank]]
        self.out = torch.empty(self.pad * self.world, dtype=torch.int32, device=device)

    def gather(self):
        dist.all_gather_into_tensor(self.out, self.buf, group=self.group)
        return self.out

    def result(self):
        return torch.cat([self.out[r * self.pad: r * self.pad + c] for r, c in enumerate(self.counts)])


def shard_d_infer(model_slice, X, argmax_fn, return_scores=False, group=None):
    """D-shard inference: `model_slice` holds this rank's columns of B and C;
    X is replicated.  All-reduce(SUM) of the N x K partial scores, then argmax."""
    S = model_slice.partial_scores(X)
    dist.all_reduce(S, op=dist.ReduceOp.SUM, group=group)
    labels = argmax_fn(S)
    return labels, (S if return_scores else None)


class DShardExchange:
    """Exchange buffers for the in-kernel D-shard reduction (hdc_model_infer_dshard).

    Allocated with torch symmetric memory (``torch.distributed._symmetric_memory``), so
    every rank's buffer is mapped into every process; the device array of the `world`
    buffer addresses is what the kernel writes through.  ``n_max`` bounds the batch
    rows (<= 32), ``K`` is the class count.  Collective: all ranks construct it together
    and then call :meth:`infer` the same number of times, each call with the same X on
    every rank (N may change from call to call: the slots are sized for 32 rows)."""

    def __init__(self, n_max, K, group=None, device=None):
        import torch.distributed._symmetric_memory as symm
        from .hdc import dshard_exchange_bytes
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        nbytes = dshard_exchange_bytes(n_max, K, self.world)
        self.n_max = n_max
        self.buf = symm.empty(nbytes // 4, dtype=torch.float32, device=dev)
        self.buf.zero_()
        handle = symm.rendezvous(self.buf, group if group is not None else dist.group.WORLD)
        self.ptrs = torch.tensor([int(p) for p in handle.buffer_ptrs], dtype=torch.int64, device=dev)
        self.epoch = 0
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)

    def infer(self, model_slice, X, return_scores=False, stream=None):
        """Labels (and scores) of X on every rank; `model_slice` holds this rank's D-slice."""
        if X.shape[0] > self.n_max:
            raise ValueError("X has %d rows, the exchange was sized for %d" % (X.shape[0], self.n_max))
        self.epoch += 1
        return model_slice.infer_dshard(X, self.ptrs, self.rank, self.world, self.epoch,
                                        return_scores=return_scores, stream=stream)
