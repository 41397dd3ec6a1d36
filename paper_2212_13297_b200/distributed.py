"""Row-sharded multi-GPU exact k-NN.

One process per GPU (torchrun, NCCL).  The dataset is split into contiguous
original-index ranges; each rank builds its own index over its shard with
``id_base`` = the shard's first original index (no communication in the
build).  Queries are replicated; every rank answers them over its shard and the
per-shard top-k (d2, id) keys are merged with ONE all-gather of B x k keys per
rank followed by the K-merge kernel (``ssb_merge_topk``).  Ids are global and
the order is the global (d2, id) order, so the answer equals a single-GPU
answer over the whole dataset.
"""

from __future__ import annotations

import numpy as np

# an empty slot (k > N): all bits set, i.e. UINT64_MAX read as unsigned -- the
# K-merge kernel's KEY_EMPTY.  Keys travel as int64 tensors (collectives have
# no uint64); every host-side ordering views them as uint64.
EMPTY = -1


def shard_range(N: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous original-index range [lo, hi) of ``rank``'s shard."""
    return rank * N // world, (rank + 1) * N // world


def pack_keys(d2, ids):
    """(d2 float32, ids int64) -> int64 keys (d2 bits << 32 | id); missing -> EMPTY.

    CUDA tensors are packed on the device by ``ssb_pack_keys`` (one kernel);
    numpy arrays and CPU tensors (the gloo tests) on the host."""
    try:
        import torch

        if isinstance(d2, torch.Tensor):
            if d2.is_cuda:
                from . import _lib
                from ._device import ptr, stream_handle

                d2c, idc = d2.contiguous(), ids.contiguous()
                keys = torch.empty(d2c.shape, dtype=torch.int64, device=d2c.device)
                _lib.call("ssb_pack_keys", ptr(d2c), ptr(idc), d2c.numel(), ptr(keys), stream_handle())
                return keys
            return torch.from_numpy(pack_keys(d2.numpy(), ids.numpy()))
    except ImportError:  # pragma: no cover
        pass
    d2 = np.ascontiguousarray(d2, np.float32)
    ids = np.asarray(ids, np.int64)
    keys = (d2.view(np.uint32).astype(np.uint64) << np.uint64(32)) | (ids & 0xFFFFFFFF).astype(np.uint64)
    keys = np.where(ids < 0, np.uint64(0xFFFFFFFFFFFFFFFF), keys)
    return keys.view(np.int64)


def unpack_keys(keys):
    """int64 (or uint64) keys -> (d2 float32, ids int64) with (inf, -1) for EMPTY (numpy)."""
    keys = np.ascontiguousarray(keys)
    u = keys.view(np.uint64) if keys.dtype == np.int64 else keys.astype(np.uint64)
    empty = u == np.uint64(0xFFFFFFFFFFFFFFFF)
    d2 = (u >> np.uint64(32)).astype(np.uint32).view(np.float32)
    ids = (u & np.uint64(0xFFFFFFFF)).astype(np.int64)
    d2 = np.where(empty, np.float32(np.inf), d2)
    ids = np.where(empty, -1, ids)
    return d2, ids


def host_merge(all_keys, k: int):
    """Host K-merge (tests, gloo): the k smallest keys of each row, unsigned order."""
    a = all_keys.numpy() if hasattr(all_keys, "numpy") else np.asarray(all_keys)
    u = np.sort(np.ascontiguousarray(a).view(np.uint64), axis=1)[:, :k]
    if u.shape[1] < k:
        pad = np.full((u.shape[0], k - u.shape[1]), np.uint64(0xFFFFFFFFFFFFFFFF))
        u = np.concatenate([u, pad], axis=1)
    return unpack_keys(u)


def gather_keys(keys, group=None):
    """All-gather every rank's (B, k) key block -> (B, world*k), rank-major."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if keys.is_cuda:
        out = torch.empty((world,) + tuple(keys.shape), dtype=keys.dtype, device=keys.device)
        dist.all_gather_into_tensor(out, keys.contiguous(), group=group)
    else:  # gloo (CPU tests)
        parts = [torch.empty_like(keys) for _ in range(world)]
        dist.all_gather(parts, keys.contiguous(), group=group)
        out = torch.stack(parts)
    return out.permute(1, 0, 2).reshape(keys.shape[0], world * keys.shape[1]).contiguous()


def merge_device(all_keys, k: int):
    """K-merge on the device: the k best of each row of (B, M) keys."""
    import torch

    from . import _lib
    from ._device import ptr, stream_handle

    B, M = all_keys.shape
    d2 = torch.empty((B, k), dtype=torch.float32, device=all_keys.device)
    ids = torch.empty((B, k), dtype=torch.int64, device=all_keys.device)
    _lib.call("ssb_merge_topk", ptr(all_keys), B, M, k, ptr(d2), ptr(ids), stream_handle())
    return d2, ids


def merge_topk(d2, ids, k: int, group=None, merge_fn=None):
    """Global top-k from every rank's shard top-k: one all-gather + K-merge.

    ``merge_fn(all_keys, k) -> (d2, ids)`` defaults to the device kernel; the
    CPU multi-process tests pass a host merge (the gloo backend has no GPU).
    """
    keys = pack_keys(d2, ids)
    all_keys = gather_keys(keys, group)
    return (merge_fn or merge_device)(all_keys, k)


class Comm:
    """The library's row-shard communicator (``ssb_comm``: NCCL inside the C
    ABI).  Rank 0 creates the NCCL id and it is broadcast over the default
    torch.distributed group; every rank then joins.  ``merge`` is the whole
    shard merge in one library call (pack -> ncclAllGather -> K-merge), and
    ``attach`` hands the communicator to this rank's index, whose query blocks
    then all-reduce (MIN) their approximate bounds across the shards."""

    ID_BYTES = 128

    def __init__(self, rank: int | None = None, world: int | None = None):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib

        self._lib = _lib
        rank = dist.get_rank() if rank is None else rank
        world = dist.get_world_size() if world is None else world
        uid = (ctypes.c_uint8 * self.ID_BYTES)()
        if rank == 0:
            _lib.call("ssb_comm_unique_id", uid)
        if world > 1:
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8,
                             device="cuda" if dist.get_backend() == "nccl" else "cpu")
            dist.broadcast(t, 0)
            uid = (ctypes.c_uint8 * self.ID_BYTES)(*t.cpu().tolist())
        self.handle = ctypes.c_void_p()
        _lib.call("ssb_comm_init", world, rank, uid, ctypes.byref(self.handle))
        self.rank, self.world = rank, world

    def merge(self, d2, ids, k: int):
        """Global (B, k) answers from this rank's (B, k) CUDA tensors."""
        import torch

        from ._device import ptr, stream_handle

        d2c, idc = d2.contiguous(), ids.contiguous()
        B = d2c.shape[0]
        out_d2 = torch.empty((B, k), dtype=torch.float32, device=d2c.device)
        out_id = torch.empty((B, k), dtype=torch.int64, device=d2c.device)
        self._lib.call("ssb_comm_merge_topk", self.handle, ptr(d2c), ptr(idc), B, k, ptr(out_d2), ptr(out_id),
                       stream_handle())
        return out_d2, out_id

    def attach(self, index):
        """Share the approximate bounds of ``index``'s query blocks across the shards."""
        si = index.index if hasattr(index, "index") else index
        self._lib.call("ssb_index_set_comm", si.handle, self.handle)

    def close(self):
        if self.handle:
            self._lib.call("ssb_comm_free", self.handle)
            self.handle = None


class ShardedIndex:
    """This rank's shard of a row-sharded index (build + query + merge)."""

    def __init__(self, data_shard, settings, id_base: int, **build_kw):
        from .build import build_index_array
        from .query import QueryEngine

        self.id_base = id_base
        self.index = build_index_array(data_shard, settings, id_base=id_base, **build_kw)
        self.engine = QueryEngine(self.index)

    def knn(self, Q, k: int, group=None):
        d2, ids, _ = self.engine.knn_device(Q, k)
        return merge_topk(d2, ids, k, group)
