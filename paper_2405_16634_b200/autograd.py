"""Differentiable winding numbers ("the Aᵀ operator is exactly the backward
function for A, which means our code also supports differentiable programming involving winding numbers").

    F = winding_number(tree, mu, width, theta)        # F_i = (A μ)_i at the tree's points (input frame)
    F.sum().backward()                                 # mu.grad = Aᵀ(∂L/∂F) through wn_eval_adjoint

Forward and backward are single libwn calls (treecode A and its adjoint); nothing is computed in Python.
With adjoint="transpose" the gradient is the exact transpose of the treecode forward at the geometry of μ
(so gradcheck-exact up to fp32), with "gather" it is the paper's own Aᵀ traversal (|s|-weighted reps).
"""
from __future__ import annotations

import torch

from . import wn


class _WindingNumber(torch.autograd.Function):
    @staticmethod
    def forward(ctx, mu, tree, width, theta, mode):
        ctx.tree, ctx.width, ctx.theta, ctx.mode = tree, width, theta, mode
        ctx.save_for_backward(mu)
        return wn.wn_eval(tree, mu.detach().contiguous(), width, theta)

    @staticmethod
    def backward(ctx, g):
        (mu,) = ctx.saved_tensors
        grad = None
        if ctx.needs_input_grad[0]:
            geom = mu.detach().contiguous() if ctx.mode == wn.WN_ADJ_TRANSPOSE else None
            grad = wn.wn_eval_adjoint(ctx.tree, g.contiguous(), ctx.width, ctx.theta, ctx.mode, geom)
        return grad, None, None, None, None


def winding_number(tree, mu: torch.Tensor, width: float, theta: float = 2.0, adjoint: str = "transpose"):
    """F = A(μ) at the tree's points, differentiable in μ."""
    mode = wn.WN_ADJ_TRANSPOSE if adjoint == "transpose" else wn.WN_ADJ_GATHER
    return _WindingNumber.apply(mu, tree, float(width), float(theta), mode)
