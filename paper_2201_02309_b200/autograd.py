"""The reconstruction as a differentiable layer: the paper
trains its dual-domain network *through* the Katsevich layer.
forward = katsevich_reconstruct, backward = katsevich_adjoint (the exact
transpose of the same linear map, checked by the dot-product test)."""
from __future__ import annotations

import torch

from .plan import Plan


class KatsevichReconstruct(torch.autograd.Function):
    """vol = A(sino) for the pitches [first_pitch, first_pitch + n_pitches);
    d loss / d sino = A^T (d loss / d vol)."""

    @staticmethod
    def forward(ctx, sino: torch.Tensor, plan: Plan, sino_first_view: int, first_pitch: int, n_pitches: int):
        ctx.plan, ctx.s0, ctx.sn = plan, sino_first_view, sino.shape[0]
        ctx.k0, ctx.np = first_pitch, n_pitches
        return plan.reconstruct(sino.detach().contiguous(), sino_first_view, first_pitch, n_pitches,
                                stream=torch.cuda.current_stream())

    @staticmethod
    def backward(ctx, grad_vol: torch.Tensor):
        g = ctx.plan.adjoint(grad_vol.detach().contiguous(), ctx.s0, ctx.sn, ctx.k0, ctx.np,
                             stream=torch.cuda.current_stream())
        return g, None, None, None, None


def reconstruct(plan: Plan, sino: torch.Tensor, sino_first_view: int, first_pitch: int = 0,
                n_pitches: int = 1) -> torch.Tensor:
    """Differentiable reconstruction: gradients flow to `sino` through the adjoint."""
    return KatsevichReconstruct.apply(sino, plan, sino_first_view, first_pitch, n_pitches)


class KatsevichReconstructBatch(torch.autograd.Function):
    """vols = A(slabs) for B independent one-pitch slabs (the paper's training workload);
    d loss / d slabs = A^T (d loss / d vols) (katsevich_adjoint_batch)."""

    @staticmethod
    def forward(ctx, slabs: torch.Tensor, plan: Plan):
        ctx.plan = plan
        return plan.reconstruct_batch(slabs.detach().contiguous(), stream=torch.cuda.current_stream())

    @staticmethod
    def backward(ctx, grad_vols: torch.Tensor):
        return ctx.plan.adjoint_batch(grad_vols.detach().contiguous(), stream=torch.cuda.current_stream()), None


def reconstruct_batch(plan: Plan, slabs: torch.Tensor) -> torch.Tensor:
    """Differentiable batch reconstruction [B][n_slab][rows][cols] -> [B][nz][ny][nx]."""
    return KatsevichReconstructBatch.apply(slabs, plan)
