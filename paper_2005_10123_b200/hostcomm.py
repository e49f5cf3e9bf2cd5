"""Host-callback collectives for rank engines (sthk_create_rank_hosted).

The engine's two multi-rank collectives -- the owner-directed exchange of the
symmetric sweep's column sums and the all-reduce of the per-block partials
 -- normally run over NCCL. `TorchDistComm` runs them through
an initialised torch.distributed process group with host tensors instead
(gloo), so several rank engines can share one GPU: the multi-GPU data flow
exercised end to end where only one device exists (tests), with the very
same planning, routes and combination as the NCCL path.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


class TorchDistComm:
    """sthk_host_comm over torch.distributed (CPU tensors: gloo)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self._torch = torch
        self._dist = dist
        self._group = group
        self.error = None
        # keep the ctypes callbacks alive as long as this object
        self._ar = _lib.ALLREDUCE_FN(self._allreduce)
        self._ex = _lib.EXCHANGE_FN(self._exchange)
        self.struct = _lib.HostCommStruct(None, self._ar, self._ex)

    def _allreduce(self, ctx, buf, count, dtype):
        try:
            ct = ctypes.c_uint64 if dtype == _lib.STHK_DTYPE_U64 else ctypes.c_double
            arr = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ct)), shape=(count,))
            if dtype == _lib.STHK_DTYPE_U64:  # two's-complement sums: int64 wraps alike
                arr = arr.view(np.int64)
            t = self._torch.from_numpy(arr)
            self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self._group)
            return 0
        except Exception as e:  # (an exception must not cross the C boundary)
            self.error = e
            return 1

    def _exchange(self, ctx, n_send, send_peer, send_buf, send_bytes, n_recv, recv_peer,
                  recv_buf, recv_bytes):
        try:
            def view(ptr, nbytes):
                a = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_uint8)),
                                          shape=(nbytes,))
                return self._torch.from_numpy(a)
            reqs = []
            for i in range(n_send):
                reqs.append(self._dist.isend(view(send_buf[i], send_bytes[i]), int(send_peer[i]),
                                             group=self._group))
            for i in range(n_recv):
                reqs.append(self._dist.irecv(view(recv_buf[i], recv_bytes[i]), int(recv_peer[i]),
                                             group=self._group))
            for r in reqs:
                r.wait()
            return 0
        except Exception as e:
            self.error = e
            return 1
