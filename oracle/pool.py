"""The fp64 oracle evaluated over independent (request, q head) units in
parallel worker processes (ORACLE — test infrastructure, SURVEY §8 c; used by
the GPU parity tests and by bench.py's cpu_baseline / --impl reference legs).

``oracle.verify_attn`` is the plain definition of the pass (§3.2); its
cost grows as L^2 per (request, head), and every (request, head) pair is an
independent problem (the paper's requests never interact, and q head h only
reads KV head h // (Hq / Hkv)).  This module only distributes those units
over host cores: each worker calls ``oracle.verify_attn`` itself on a
one-request, one-head slice, so no arithmetic is added or reordered.

Workers come from a fresh single-threaded fork server (never forked from the
multi-threaded test process), read the inputs from POSIX shared memory and
run single-threaded BLAS, so the pool uses one core per worker.  They never
touch CUDA or torch.
"""

from __future__ import annotations

import concurrent.futures as cf
import multiprocessing as mp
import os
from multiprocessing import shared_memory
from typing import Optional, Sequence

import numpy as np

from .attention import verify_attn
from .mask import visible_mask

_G: dict = {}
_SHM: list = []


def _init_worker(arrays: dict, scalars: dict):
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # pragma: no cover
        pass
    for name, (shm_name, shape, dtype) in arrays.items():
        shm = shared_memory.SharedMemory(name=shm_name)
        _SHM.append(shm)
        _G[name] = np.ndarray(shape, dtype=dtype, buffer=shm.buf)
    _G.update(scalars)


def _unit(args):
    b, h = args
    g = _G
    r = g["q"].shape[2] // g["k"].shape[2]
    kv = h // r
    q = g["q"][b:b + 1, :, h:h + 1]
    k = g["k"][b:b + 1, :, kv:kv + 1]
    v = g["v"][b:b + 1, :, kv:kv + 1]
    bnd = g["bnd"][b]
    O, LSE = verify_attn(q, k, v, g["N"], g["K"], g["S"], bnd, tree_parent=g["tree"], scale=g["scale"],
                                row_chunk=g["row_chunk"])
    return b, h, O[0, :, 0].astype(np.float64), LSE[0, 0]


def available_workers(per_worker_gb: float) -> int:
    cpus = os.cpu_count() or 1
    try:
        with open("/proc/meminfo") as f:
            avail_kb = next(int(ln.split()[1]) for ln in f if ln.startswith("MemAvailable"))
        by_mem = int(avail_kb / 1e6 * 0.6 / max(per_worker_gb, 0.05))
    except Exception:  # pragma: no cover
        by_mem = cpus
    return max(1, min(cpus, by_mem))


def pool_map(fn, units, shared: dict, per_worker_gb: float, workers: Optional[int] = None):
    """Yield fn(unit) for every unit (any order), computed by single-threaded
    worker processes that see ``shared`` as the module global ``_G`` (numpy
    arrays through shared memory, everything else pickled once)."""
    n_workers = workers or available_workers(per_worker_gb)
    n_workers = max(1, min(n_workers, len(units)))
    if n_workers == 1:
        _G.update(shared)
        try:
            yield from map(fn, units)
        finally:
            _G.clear()
        return
    segs, arrays, scalars = [], {}, {}
    try:
        for name, val in shared.items():
            if isinstance(val, np.ndarray):
                val = np.ascontiguousarray(val)
                shm = shared_memory.SharedMemory(create=True, size=max(1, val.nbytes))
                segs.append(shm)
                np.ndarray(val.shape, dtype=val.dtype, buffer=shm.buf)[...] = val
                arrays[name] = (shm.name, val.shape, val.dtype.str)
            else:
                scalars[name] = val
        # a process pool that fails loudly (BrokenProcessPool) if a worker
        # dies, e.g. when the caller's __main__ cannot be re-imported
        ctx = mp.get_context("forkserver")
        with cf.ProcessPoolExecutor(n_workers, mp_context=ctx, initializer=_init_worker,
                                    initargs=(arrays, scalars)) as ex:
            futs = [ex.submit(fn, u) for u in units]
            for f in cf.as_completed(futs):
                yield f.result()
    finally:
        for shm in segs:
            shm.close()
            shm.unlink()


def host_f32(x) -> np.ndarray:
    """Host copy of an input: bf16 values are exact in fp32; fp64 inputs (the
    FP8 tests' dequantised x8 * descale) stay fp64."""
    if hasattr(x, "detach"):
        import torch
        x = x.detach().to("cpu")
        x = (x if x.dtype == torch.float64 else x.float()).numpy()
    return np.ascontiguousarray(x)


def verify_attn_parallel(q, k, v, N: int, K: int, S: int, boundaries, tree_parent=None,
                         scale: Optional[float] = None, batches: Optional[Sequence[int]] = None,
                         heads: Optional[Sequence[int]] = None, workers: Optional[int] = None):
    """Same result as ``oracle.verify_attn`` (O [nb, L, nh, d], LSE [nb, nh, L]
    fp64), computed by a pool of processes over (request, head) units."""
    qn, kn, vn = host_f32(q), host_f32(k), host_f32(v)
    B, L, Hq, d = qn.shape
    bnd = np.asarray(boundaries, dtype=np.int64)
    if bnd.ndim == 1:
        bnd = np.broadcast_to(bnd, (B, K))
    batches = list(range(B)) if batches is None else list(batches)
    heads = list(range(Hq)) if heads is None else list(heads)
    row_chunk = 1024
    per_worker_gb = 5 * row_chunk * L * 8 / 1e9 + 3 * L * d * 8 / 1e9 + L * L / 1e9
    units = [(b, h) for b in batches for h in heads]
    O = np.zeros((len(batches), L, len(heads), vn.shape[3]))
    LSE = np.zeros((len(batches), len(heads), L))
    bi = {b: i for i, b in enumerate(batches)}
    hi = {h: i for i, h in enumerate(heads)}
    shared = dict(q=qn, k=kn, v=vn, bnd=bnd, N=N, K=K, S=S, tree=tree_parent, scale=scale, row_chunk=row_chunk)
    for b, h, o, lse in pool_map(_unit, units, shared, per_worker_gb, workers):
        O[bi[b], :, hi[h]] = o
        LSE[bi[b], hi[h]] = lse
    return O, LSE

