"""B200-native k-split multi-lane allreduce (arXiv 2508.13397).

Thin Python binding over the C ABI in ``include/lane_allreduce.h``
(liblane_allreduce.so, sm_100a). PyTorch is used for device memory, streams
and the one-time IPC handle exchange (``torch.distributed``); every step of
the allreduce runs in the library's CUDA kernels.

    comm = LaneComm(nodes=2, gpus_per_node=4, procs_per_gpu=1)   # under torchrun
    comm.allreduce(out, inp)                                      # out = sum over ranks

    emu = LaneEmulator(2, 4, 1)          # all 8 ranks on one GPU (same kernels)
    emu.allreduce(outs, inps)
"""
from __future__ import annotations

import ctypes

from . import _lib
from ._lib import DTYPE, HANDLE_BYTES, LaneError

__all__ = ["LaneComm", "LaneEmulator", "LaneError", "topology", "partition_units", "version"]


def _torch():
    import torch
    return torch


_DTYPE_MAP = None


def _dtype_code(t) -> int:
    global _DTYPE_MAP
    if _DTYPE_MAP is None:  # built once: the per-call path stays a dict lookup
        torch = _torch()
        _DTYPE_MAP = {torch.int32: DTYPE["int32"], torch.float32: DTYPE["float32"],
                      torch.bfloat16: DTYPE["bfloat16"]}
    code = _DTYPE_MAP.get(t.dtype)
    if code is None:
        raise LaneError(-2, f"dtype: {t.dtype} is not supported (int32, float32, bfloat16)")
    return code


def _check_dev_tensor(t, device_index: int, what: str):
    if not t.is_cuda or t.device.index != device_index:
        raise LaneError(-1, f"{what}: must be a CUDA tensor on device {device_index}")
    if not t.is_contiguous():
        raise LaneError(-1, f"{what}: must be contiguous")


def _check_host_tensor(t, what: str):
    if t.is_cuda:
        raise LaneError(-1, f"{what}: must be a host (CPU) tensor")
    if not t.is_contiguous():
        raise LaneError(-1, f"{what}: must be contiguous")


def _check_pair(out, inp, op: str, host: bool = False, device_index: int = 0):
    """The one argument check of every allreduce entry point: op, placement,
    contiguity, and out matching inp in numel and dtype (the C ABI copies
    count * itemsize bytes into every output)."""
    if op != "sum":
        raise LaneError(-2, "op: only 'sum' (MPI_SUM)")
    for t, what in ((inp, "inp"), (out, "out")):
        if host:
            _check_host_tensor(t, what)
        else:
            _check_dev_tensor(t, device_index, what)
    if out.numel() != inp.numel() or out.dtype != inp.dtype:
        raise LaneError(-1, "out: must match inp in numel and dtype")


def _stream_handle(stream, device_index=None) -> int:
    """Raw cudaStream_t of ``stream`` (default: the current stream of
    ``device_index``, read without building a torch.cuda.Stream object —
    the per-call host cost matters for small messages)."""
    torch = _torch()
    if stream is not None:
        return int(stream.cuda_stream)
    if device_index is not None:
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if raw is not None:
            return int(raw(device_index))
    return int(torch.cuda.current_stream().cuda_stream)


def version() -> str:
    return _lib.load().lane_allreduce_version().decode()


def topology(nodes: int, gpus_per_node: int, rank: int):
    """(node, gpu, comm_group ranks, comm_lane ranks) of ``rank`` — host only."""
    lib = _lib.load()
    node, gpu = ctypes.c_int(), ctypes.c_int()
    grp = (ctypes.c_int * max(gpus_per_node, 1))()
    lane = (ctypes.c_int * max(nodes, 1))()
    _lib.check(lib.lane_topology_query(nodes, gpus_per_node, rank, ctypes.byref(node), ctypes.byref(gpu),
                                       grp, lane))
    return node.value, gpu.value, list(grp)[:gpus_per_node], list(lane)[:nodes]


def partition_units(count: int, itemsize: int, nodes: int, gpus_per_node: int, procs_per_gpu: int,
                    chunk_granules: int = 0, round_granules: int = 0):
    """The library's ownership units (host only): list of 9-tuples
    (round, l, c, g, a, part_start, part_end, start, end)."""
    lib = _lib.load()
    n = ctypes.c_uint64()
    _lib.check(lib.lane_partition_query(count, itemsize, nodes, gpus_per_node, procs_per_gpu,
                                        chunk_granules, round_granules, None, 0, ctypes.byref(n)))
    buf = (ctypes.c_int64 * (9 * max(n.value, 1)))()
    _lib.check(lib.lane_partition_query(count, itemsize, nodes, gpus_per_node, procs_per_gpu,
                                        chunk_granules, round_granules, buf, n.value, ctypes.byref(n)))
    flat = list(buf)
    return [tuple(flat[9 * i:9 * i + 9]) for i in range(n.value)]


class _CommBase:
    _comm = None

    def plan(self, count: int, dtype: str = "float32", algorithm: str = "lane") -> dict:
        """Launch plan of ``allreduce`` (algorithm="lane") or ``allreduce_ring``
        ("ring"): chunk / round granules, CTAs per CTA group, launches."""
        lib = _lib.load()
        cg, rg = ctypes.c_int64(), ctypes.c_int64()
        C, launches = ctypes.c_int(), ctypes.c_int()
        fn = lib.lane_allreduce_ring_plan if algorithm == "ring" else lib.lane_allreduce_plan
        _lib.check(fn(self._comm, count, DTYPE[dtype], ctypes.byref(cg), ctypes.byref(rg),
                      ctypes.byref(C), ctypes.byref(launches)), self._comm)
        return {"chunk_granules": cg.value, "round_granules": rg.value, "ctas_per_group": C.value,
                "launches": launches.value}

    def ring_protocol(self, count: int, dtype: str = "float32") -> str:
        """'ll' or 'll128': the protocol a ring allreduce (Alg. 1) call of this size uses."""
        pr = ctypes.c_int()
        _lib.check(_lib.load().lane_allreduce_ring_protocol(self._comm, count, DTYPE[dtype], ctypes.byref(pr)),
                   self._comm)
        return {1: "ll", 2: "ll128"}.get(pr.value, "simple")

    def protocol(self, count: int, dtype: str = "float32") -> str:
        """'ll', 'll128' or 'simple': the signalling protocol a call of this size uses."""
        pr = ctypes.c_int()
        _lib.check(_lib.load().lane_allreduce_protocol(self._comm, count, DTYPE[dtype], ctypes.byref(pr)),
                   self._comm)
        return {1: "ll", 2: "ll128"}.get(pr.value, "simple")

    TRACE_FIELDS = ("prod_total", "prod_flag_wait", "prod_empty_wait", "prod_tiles", "store_total",
                    "store_full_wait", "store_sync", "store_read_wait", "store_flush", "store_jobs",
                    "phase_A", "phase_B", "phase_C", "phase_D", "phase_E", "bytes_stored",
                    "start_abs", "enter_wait", "end_abs", "smid", "entry_abs")

    def trace(self) -> list:
        """Per-CTA stall accounting of the last launch (needs LANE_TRACE=1 at
        construction): list of dicts, nanoseconds."""
        lib = _lib.load()
        n = ctypes.c_size_t()
        _lib.check(lib.lane_allreduce_trace(self._comm, None, 0, ctypes.byref(n)), self._comm)
        buf = (ctypes.c_uint64 * max(n.value, 1))()
        _lib.check(lib.lane_allreduce_trace(self._comm, buf, n.value, ctypes.byref(n)), self._comm)
        w = len(self.TRACE_FIELDS)
        return [dict(zip(self.TRACE_FIELDS, list(buf)[i * w:(i + 1) * w])) for i in range(n.value // w)]

    def check(self) -> None:
        _lib.check(_lib.load().lane_allreduce_check(self._comm), self._comm)

    def close(self) -> None:
        if self._comm is not None:
            _lib.load().lane_allreduce_finalize(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LaneComm(_CommBase):
    """One rank of a multi-GPU lane allreduce (one process per GPU).

    ``nodes * gpus_per_node`` must equal the world size; rank ``p`` is
    virtual node ``p // gpus_per_node``, GPU ``p % gpus_per_node``. The IPC
    handles are all-gathered through ``torch.distributed`` (``group``, default
    world) once, at construction — the only host-side collective."""

    def __init__(self, nodes: int, gpus_per_node: int, procs_per_gpu: int = 1, *, rank=None,
                 device=None, group=None):
        torch = _torch()
        import torch.distributed as dist
        lib = _lib.load()
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        if device is None:
            device = torch.cuda.current_device()
        self.nodes, self.gpus_per_node, self.procs_per_gpu = nodes, gpus_per_node, procs_per_gpu
        self.rank, self.device = rank, device
        h = ctypes.c_void_p()
        code = lib.lane_allreduce_init_rank(nodes, gpus_per_node, procs_per_gpu, rank, device, ctypes.byref(h))
        _lib.check(code, None)
        self._comm = h
        blob = ctypes.create_string_buffer(HANDLE_BYTES)
        size = ctypes.c_size_t()
        _lib.check(lib.lane_allreduce_get_handle(self._comm, blob, ctypes.byref(size)), self._comm)
        blobs = exchange_blobs(bytes(blob.raw[:size.value]), group)
        if len(blobs) != nodes * gpus_per_node:
            raise LaneError(-1, f"world size {len(blobs)} != nodes*gpus_per_node {nodes * gpus_per_node}")
        allb = b"".join(blobs)
        _lib.check(lib.lane_allreduce_open_peers(self._comm, allb, size.value), self._comm)

    def allreduce(self, out, inp, op: str = "sum", stream=None):
        """out[i] = sum over ranks of inp[i]; enqueued on ``stream`` (default:
        current). ``out is inp`` (same storage) is in-place."""
        _check_pair(out, inp, op, device_index=self.device)
        code = _lib.load().lane_allreduce(self._comm, inp.data_ptr(), out.data_ptr(), inp.numel(),
                                          _dtype_code(inp), 0, _stream_handle(stream, self.device))
        _lib.check(code, self._comm)
        return out

    def allreduce_ring(self, out, inp, op: str = "sum", stream=None):
        """The paper's "standard" ring allreduce (Alg. 1; with k > 1 the
        standard multi-PPG approach): same contract as ``allreduce``, ring
        reduction order with per-hop rounding."""
        _check_pair(out, inp, op, device_index=self.device)
        code = _lib.load().lane_allreduce_ring(self._comm, inp.data_ptr(), out.data_ptr(), inp.numel(),
                                               _dtype_code(inp), 0, _stream_handle(stream, self.device))
        _lib.check(code, self._comm)
        return out

    def allreduce_approach2(self, out, inp, op: str = "sum", stream=None):
        """The paper's draft "approach 2" (node allreduce, then lane allreduce
        of the whole buffer): same results as ``allreduce``, more traffic."""
        _check_pair(out, inp, op, device_index=self.device)
        code = _lib.load().lane_allreduce_approach2(self._comm, inp.data_ptr(), out.data_ptr(), inp.numel(),
                                                    _dtype_code(inp), 0, _stream_handle(stream, self.device))
        _lib.check(code, self._comm)
        return out

    def register(self, t, group=None) -> int:
        """Collective: register CUDA tensor ``t`` for zero-copy allreduce (every
        rank registers its own buffer of the same size, in the same order).
        Allreduces on tensors inside registered buffers then read peers'
        sendbufs and write peers' recvbufs directly (P L330 IPC sharing)."""
        _check_dev_tensor(t, self.device, "t")
        lib = _lib.load()
        blob = ctypes.create_string_buffer(HANDLE_BYTES)
        size = ctypes.c_size_t()
        nbytes = t.numel() * t.element_size()
        _lib.check(lib.lane_allreduce_register_handle(self._comm, t.data_ptr(), nbytes, blob, ctypes.byref(size)),
                   self._comm)
        blobs = exchange_blobs(bytes(blob.raw[:size.value]), group)
        rid = ctypes.c_int()
        _lib.check(lib.lane_allreduce_register_open(self._comm, b"".join(blobs), size.value, ctypes.byref(rid)),
                   self._comm)
        return rid.value

    def deregister(self, reg_id: int) -> None:
        _lib.check(_lib.load().lane_allreduce_deregister(self._comm, reg_id), self._comm)

    def allreduce_host(self, out_host, inp_host, op: str = "sum", stream=None):
        """End-to-end allreduce of HOST tensors (H2D, kernels, D2H on one
        stream). Synchronizes the stream before returning."""
        torch = _torch()
        _check_pair(out_host, inp_host, op, host=True)
        code = _lib.load().lane_allreduce_host(self._comm, inp_host.data_ptr(), out_host.data_ptr(),
                                               inp_host.numel(), _dtype_code(inp_host), 0,
                                               _stream_handle(stream, self.device))
        _lib.check(code, self._comm)
        (stream or torch.cuda.current_stream(self.device)).synchronize()
        return out_host


def exchange_blobs(blob: bytes, group=None) -> list[bytes]:
    """All-gather one opaque blob per rank, in rank order (IPC handle
    broadcast, P L330). Uses torch.distributed; works on gloo and nccl."""
    import torch.distributed as dist
    if not dist.is_initialized():
        return [blob]
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


class LaneEmulator(_CommBase):
    """All ``nodes * gpus_per_node`` ranks on ONE GPU: the same kernels and the
    same cross-rank flag protocol, run as one cooperative launch."""

    def __init__(self, nodes: int, gpus_per_node: int, procs_per_gpu: int = 1, device=None):
        torch = _torch()
        lib = _lib.load()
        if device is None:
            device = torch.cuda.current_device()
        self.nodes, self.gpus_per_node, self.procs_per_gpu = nodes, gpus_per_node, procs_per_gpu
        self.P = nodes * gpus_per_node
        self.device = device
        h = ctypes.c_void_p()
        _lib.check(lib.lane_allreduce_init_emulated(nodes, gpus_per_node, procs_per_gpu, device, ctypes.byref(h)),
                   None)
        self._comm = h

    def _ptrs(self, ts, what, dev=True):
        if len(ts) != self.P:
            raise LaneError(-1, f"{what}: need {self.P} tensors, got {len(ts)}")
        for i, t in enumerate(ts):
            if dev:
                _check_dev_tensor(t, self.device, f"{what}[{i}]")
            else:
                _check_host_tensor(t, f"{what}[{i}]")
        return (ctypes.c_void_p * self.P)(*[t.data_ptr() for t in ts])

    def _args(self, outs, inps, op, dev=True):
        """Checks shared by every emulated entry point; returns the ctypes
        argument tuple (sendbufs, recvbufs, count, dtype)."""
        if op != "sum":
            raise LaneError(-2, "op: only 'sum' (MPI_SUM)")
        n = inps[0].numel()
        if any(t.numel() != n or t.dtype != inps[0].dtype for t in list(inps) + list(outs)):
            raise LaneError(-1, "all tensors must have the same numel and dtype")
        return self._ptrs(inps, "inps", dev), self._ptrs(outs, "outs", dev), n, _dtype_code(inps[0])

    def allreduce(self, outs, inps, op: str = "sum", stream=None):
        code = _lib.load().lane_allreduce_emulated(self._comm, *self._args(outs, inps, op), 0,
                                                   _stream_handle(stream, self.device))
        _lib.check(code, self._comm)
        return outs

    def allreduce_ring(self, outs, inps, op: str = "sum", stream=None):
        """Ring allreduce (Alg. 1) of all emulated ranks."""
        code = _lib.load().lane_allreduce_ring_emulated(self._comm, *self._args(outs, inps, op), 0,
                                                        _stream_handle(stream, self.device))
        _lib.check(code, self._comm)
        return outs

    def allreduce_approach2(self, outs, inps, op: str = "sum", stream=None):
        """'Approach 2' (node allreduce, then lane allreduce) of all emulated ranks."""
        code = _lib.load().lane_allreduce_approach2_emulated(self._comm, *self._args(outs, inps, op), 0,
                                                             _stream_handle(stream, self.device))
        _lib.check(code, self._comm)
        return outs

    def allreduce_host(self, outs_host, inps_host, op: str = "sum", stream=None):
        torch = _torch()
        code = _lib.load().lane_allreduce_emulated_host(self._comm, *self._args(outs_host, inps_host, op, dev=False),
                                                        0, _stream_handle(stream, self.device))
        _lib.check(code, self._comm)
        (stream or torch.cuda.current_stream(self.device)).synchronize()
        return outs_host
