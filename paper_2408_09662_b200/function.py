"""PyTorch-facing API: call a tape on batched CUDA tensors.

``Function(tape)(x0, x1, ...)`` takes one ``[batch, nnz_in[i]]`` tensor per
input (env-major, the reference workspace layout) and returns one
``[batch, nnz_out[j]]`` tensor per output, computed on the tensors' device
on torch's current stream.  ``layout="soa"`` takes/returns ``[nnz, batch]``
tensors instead (every load/store coalesced without staging).  This is the
"host-ML-framework tensor interface" the paper describes (§III.B)
and the reference scopes out.
"""

from __future__ import annotations

import torch

from .plan import get_plan
from .tape import as_tape

__all__ = ["Function"]


class Function:
    def __init__(self, tape, *, dtype=torch.float64, layout: str = "aos", **plan_options):
        if dtype not in (torch.float64, torch.float32):
            raise ValueError(f"dtype must be torch.float64 or torch.float32, got {dtype}")
        if layout not in ("aos", "soa"):
            raise ValueError(f"layout must be 'aos' or 'soa', got {layout!r}")
        self.tape = as_tape(tape)
        self.dtype = dtype
        self.layout = layout
        self.plan = get_plan(self.tape, dtype="float32" if dtype == torch.float32 else "float64", **plan_options)

    @property
    def nnz_in(self):
        return self.tape.nnz_in

    @property
    def nnz_out(self):
        return self.tape.nnz_out

    def _check(self, inputs):
        t = self.tape
        if len(inputs) != t.n_in:
            raise ValueError(f"expected {t.n_in} inputs, got {len(inputs)}")
        batch = None
        device = None
        for i, x in enumerate(inputs):
            if not isinstance(x, torch.Tensor):
                raise TypeError(f"input {i}: expected a torch.Tensor, got {type(x).__name__}")
            if x.dtype != self.dtype:
                raise ValueError(f"input {i}: dtype {x.dtype} != {self.dtype}")
            if not x.is_cuda:
                raise ValueError(f"input {i}: tensor must live on a CUDA device")
            if x.dim() != 2:
                raise ValueError(f"input {i}: expected a 2-D tensor, got shape {tuple(x.shape)}")
            nz, b = (x.shape[1], x.shape[0]) if self.layout == "aos" else (x.shape[0], x.shape[1])
            if nz != t.nnz_in[i]:
                raise ValueError(f"input {i}: expected {t.nnz_in[i]} nonzeros, got shape {tuple(x.shape)}")
            if batch is None:
                batch, device = b, x.device
            elif b != batch or x.device != device:
                raise ValueError(f"input {i}: batch/device differs from input 0")
        return batch, device

    def _check_out(self, out, b, dev):
        """Caller-provided outputs are written through raw pointers: check count, shape,
        dtype, device and layout exactly (a mismatch would be an out-of-bounds write)."""
        t = self.tape
        out = list(out)
        if len(out) != t.n_out:
            raise ValueError(f"out: expected {t.n_out} tensors, got {len(out)}")
        for j, o in enumerate(out):
            if not isinstance(o, torch.Tensor):
                raise TypeError(f"out {j}: expected a torch.Tensor, got {type(o).__name__}")
            want = (b, t.nnz_out[j]) if self.layout == "aos" else (t.nnz_out[j], b)
            if tuple(o.shape) != want:
                raise ValueError(f"out {j}: expected shape {want}, got {tuple(o.shape)}")
            if o.dtype != self.dtype:
                raise ValueError(f"out {j}: dtype {o.dtype} != {self.dtype}")
            if o.device != dev:
                raise ValueError(f"out {j}: device {o.device} != {dev}")
            if o.numel() == 0:
                continue
            if self.layout == "aos" and not o.is_contiguous():
                raise ValueError(f"out {j}: an AoS output must be contiguous")
            if self.layout == "soa" and o.shape[1] > 1 and o.stride(1) != 1:
                raise ValueError(f"out {j}: an SoA output needs unit stride along the batch")
        if self.layout == "soa":
            lds = {o.stride(0) for o in out if o.shape[0] > 1 and o.numel()}
            if len(lds) > 1:
                raise ValueError(f"out: SoA outputs must share one leading dimension, got {sorted(lds)}")
        return out

    def __call__(self, *inputs, out=None, batch: int | None = None, device=None):
        t = self.tape
        if t.n_in:
            b, dev = self._check(inputs)
        else:
            if batch is None:
                raise ValueError("tape has no inputs: pass batch=")
            b, dev = int(batch), torch.device(device if device is not None else "cuda")
            if dev.type == "cuda" and dev.index is None:
                dev = torch.device("cuda", torch.cuda.current_device())
        if out is not None:
            out = self._check_out(out, b, dev)
        if self.layout == "aos":
            inputs = [x.contiguous() for x in inputs]
            outs = out if out is not None else [torch.empty((b, nz), dtype=self.dtype, device=dev) for nz in t.nnz_out]
        else:
            inputs = [x if (x.shape[1] <= 1 or x.stride(1) == 1) else x.contiguous() for x in inputs]
            outs = out if out is not None else [torch.empty((nz, b), dtype=self.dtype, device=dev) for nz in t.nnz_out]
        if b == 0:
            return outs
        stream = torch.cuda.current_stream(dev).cuda_stream
        if self.layout == "aos":
            self.plan.eval_device_ptrs([x.data_ptr() for x in inputs], [o.data_ptr() for o in outs], 0, b,
                                       dev.index or 0, stream)
        else:
            # one leading dimension for every row: the outputs' (caller-fixed) if given, else
            # the inputs' common stride, else b; inputs off that stride are re-laid out
            out_lds = {o.stride(0) for o in outs if o.shape[0] > 1}
            in_lds = {x.stride(0) for x in inputs if x.shape[0] > 1}
            if out is not None and out_lds:
                ld = out_lds.pop()
            elif len(in_lds) == 1 and (not out_lds or out_lds == in_lds):
                ld = in_lds.pop()
            else:
                ld = b
            if ld < b:
                raise ValueError(f"SoA leading dimension {ld} < batch {b}")
            fixed = []
            for x in inputs:
                if x.shape[0] > 1 and x.stride(0) != ld:
                    y = torch.empty_strided(tuple(x.shape), (ld, 1), dtype=x.dtype, device=x.device)
                    y.copy_(x)
                    x = y
                fixed.append(x)
            self.plan.eval_device_soa([x.data_ptr() for x in fixed], [o.data_ptr() for o in outs], ld, 0, b,
                                      dev.index or 0, stream)
        return outs
