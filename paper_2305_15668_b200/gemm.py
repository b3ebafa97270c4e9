"""Grouped tcgen05 GEMM with fused epilogues (csrc/gemm_tc.cu, `fedhc_gemm`).

The client-model building block for models beyond the reference's linear
model: D_g = epilogue(A_g . B_g^T) with bf16 operands in either K-major or
MN-major storage, so forward, dgrad and wgrad all run without transposes.

    A: [G, M, K] (a_mn=False) or [G, K, M] (a_mn=True), bf16, contiguous
    B: [G, N, K] (b_mn=False) or [G, K, N] (b_mn=True), bf16, contiguous
    M % 64 == 0 (M=64 tiles run the UMMA M=64 shape), N % 32 == 0 (N % 64 == 0
    when b_mn), K % 64 == 0.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _abi
from ._abi import EPI_BF16, EPI_BIAS_RELU_BF16, EPI_F32, EPI_RELU_MASK_BF16, EPI_SGD  # noqa: F401


def _dims(A: torch.Tensor, B: torch.Tensor, a_mn: bool, b_mn: bool):
    if A.dtype != torch.bfloat16 or B.dtype != torch.bfloat16:
        raise TypeError("gemm operands must be bf16")
    if A.dim() == 2:
        A = A.unsqueeze(0)
    if B.dim() == 2:
        B = B.unsqueeze(0)
    if not (A.is_contiguous() and B.is_contiguous()):
        raise ValueError("gemm operands must be contiguous")
    G = A.shape[0]
    if B.shape[0] != G:
        raise ValueError("group counts differ")
    K, M = (A.shape[1], A.shape[2]) if a_mn else (A.shape[2], A.shape[1])
    Kb, N = (B.shape[1], B.shape[2]) if b_mn else (B.shape[2], B.shape[1])
    if Kb != K:
        raise ValueError(f"inner dimensions differ: {K} vs {Kb}")
    return A, B, G, M, N, K


def gemm(A: torch.Tensor, B: torch.Tensor, *, a_mn: bool = False, b_mn: bool = False, epilogue: int = EPI_F32,
         out: torch.Tensor | None = None, bias: torch.Tensor | None = None, bias_per_row: bool = False,
         master: torch.Tensor | None = None, shadow: torch.Tensor | None = None, lr: float = 0.0,
         mask: torch.Tensor | None = None, rowsum: torch.Tensor | None = None,
         stream: int | None = None) -> torch.Tensor | None:
    """Launch one grouped GEMM; returns the output tensor (the master for EPI_SGD)."""
    A, B, G, M, N, K = _dims(A, B, a_mn, b_mn)
    args = _abi.GemmArgs(G=G, M=M, N=N, K=K, a_mn=int(a_mn), b_mn=int(b_mn), A=A.data_ptr(), B=B.data_ptr(),
                         epilogue=epilogue, bias_per_row=int(bias_per_row))
    keep = [A, B]
    if epilogue == EPI_SGD:
        if master is None or master.dtype != torch.float32 or master.numel() != G * M * N:
            raise ValueError("EPI_SGD needs an fp32 master of G*M*N elements")
        args.master, args.lr = master.data_ptr(), float(lr)
        if shadow is not None:
            if shadow.dtype != torch.bfloat16 or shadow.numel() != G * M * N:
                raise ValueError("shadow must be bf16 with G*M*N elements")
            args.shadow = shadow.data_ptr()
        result = master
    else:
        dt = torch.float32 if epilogue == EPI_F32 else torch.bfloat16
        if out is None:
            out = torch.empty(G, M, N, dtype=dt, device=A.device)
        elif out.dtype != dt or out.numel() != G * M * N or not out.is_contiguous():
            raise ValueError("out has the wrong dtype/shape")
        args.D = out.data_ptr()
        if epilogue == EPI_BIAS_RELU_BF16:
            if bias is None or bias.dtype != torch.float32:
                raise ValueError("EPI_BIAS_RELU_BF16 needs an fp32 bias")
            per = M if bias_per_row else N
            if bias.numel() not in (per, G * per):
                raise ValueError("bias must hold M (per-row) or N (per-column) values, optionally per group")
            args.bias = bias.data_ptr()
            args.bias_gstride = per if bias.numel() == G * per else 0
            keep.append(bias)
        if epilogue == EPI_RELU_MASK_BF16:
            if mask is None or mask.dtype != torch.bfloat16 or mask.numel() != G * M * N:
                raise ValueError("EPI_RELU_MASK_BF16 needs a bf16 mask shaped like the output")
            args.mask = mask.data_ptr()
        if rowsum is not None:
            if rowsum.dtype != torch.float32 or rowsum.numel() != G * M:
                raise ValueError("rowsum must be fp32 with G*M elements")
            args.rowsum = rowsum.data_ptr()
        result = out
    s = torch.cuda.current_stream().cuda_stream if stream is None else stream
    _abi.check(_abi.lib.fedhc_gemm(C.byref(args), s))
    return result
