"""(e) Offloaded embedding: the full embedding table stays in pinned host
memory (memory_report's embedding_bytes_gpu == 0, head.cpp:219-237) and the
prompt's rows are fetched per request, either by a zero-copy kernel reading
host memory over the link or by one staged cudaMemcpyAsync on a side stream
(the transfer the reference only models in offload_sim.cpp:44-60)."""
from __future__ import annotations

import numpy as np
import torch

from ._lib import SVT_F32, call
from .tailored_head import _stream, torch_dtype


class HostEmbedding:
    def __init__(self, table: np.ndarray, storage: int = SVT_F32):
        t = torch.from_numpy(np.ascontiguousarray(table, np.float32))
        self.rows, self.dim = t.shape
        self.storage = storage
        self.table = t.to(torch_dtype(storage)).pin_memory()
        self._staging = None

    def lookup(self, ids, mode: str = "zero_copy", stream=None) -> torch.Tensor:
        ids = np.ascontiguousarray(np.asarray(ids, np.uint32))
        n = ids.size
        out = torch.empty((max(n, 1), self.dim), dtype=self.table.dtype, device="cuda")
        if mode == "zero_copy":
            d_ids = torch.from_numpy(ids.view(np.int32) if n else np.zeros(1, np.int32)).cuda()
            bad = torch.zeros(1, dtype=torch.int32, device="cuda")
            call("svt_embed_lookup_zero_copy", self.table.data_ptr(), self.storage, self.rows,
                 self.dim, d_ids.data_ptr(), n, out.data_ptr(), bad.data_ptr(), _stream(stream))
            if int(bad.item()):
                from ._lib import IntegrityError
                raise IntegrityError("token id out of range for the embedding table")
        elif mode == "staged":
            need = max(n, 1) * self.dim
            if self._staging is None or self._staging.numel() < need:
                self._staging = torch.empty(need, dtype=self.table.dtype).pin_memory()
            call("svt_embed_lookup_staged", self.table.data_ptr(), self.storage, self.rows,
                 self.dim, ids.ctypes.data if n else None, n, self._staging.data_ptr(),
                 out.data_ptr(), _stream(stream))
        else:
            raise ValueError(mode)
        return out[:n]
