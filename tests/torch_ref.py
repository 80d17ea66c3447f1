"""Autograd reference for render_backward (TEST INFRASTRUCTURE).

A float64 PyTorch restatement of the reference's per-pixel renderer
(render_reference, render.hpp:360-408: every pixel walks all depth-sorted
visible splats whose tile span holds it) with project (render.hpp:104-174) and
splat_alpha (render.hpp:189-231) written as differentiable expressions.  The
hard gates of the reference (alpha floor, 0.99 cap, colour clamp, the
transmittance break) are the same piecewise definitions, so autograd yields
exactly the gradients render_backward's formulas intend; the oracle's float
backward is checked against it at a relative tolerance.  Small scenes only.
"""
from __future__ import annotations

import math

import numpy as np
import torch

SH0 = 0.28209479177387814
SH1 = 0.4886025119029199
SH2 = [1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792, 0.5462742152960396]
SH3 = [-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154, -0.4570457994644658,
       1.445305721320277, -0.5900435899266435]


def sh_basis(d):
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    xx, yy, zz = x * x, y * y, z * z
    one = torch.ones_like(x)
    return torch.stack([
        SH0 * one, -SH1 * y, SH1 * z, -SH1 * x,
        SH2[0] * x * y, SH2[1] * y * z, SH2[2] * (2 * zz - xx - yy), SH2[3] * x * z, SH2[4] * (xx - yy),
        SH3[0] * y * (3 * xx - yy), SH3[1] * x * y * z, SH3[2] * y * (4 * zz - xx - yy),
        SH3[3] * z * (2 * zz - 3 * xx - 3 * yy), SH3[4] * x * (4 * zz - xx - yy), SH3[5] * z * (xx - yy),
        SH3[6] * x * (xx - 3 * yy)], 1)


def render(params, cam, exposure=None):
    """params: dict of float64 tensors mean (n,3), scale (n,3), rot (n,4 wxyz), sh (n,48), falloff, parent_falloff,
    t (n,), inv_k (n,) (constant).  Returns exposed colour (3,H,W) and inverse depth (H,W)."""
    W = torch.tensor(np.asarray(cam.world_to_camera, np.float64))
    R, tr = W[:, :3], W[:, 3]
    fx, fy, cx, cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    w, h = int(cam.width), int(cam.height)
    mean, scale, rot = params["mean"], params["scale"], params["rot"]
    n = mean.shape[0]
    tc = mean @ R.T + tr
    q = rot / rot.norm(dim=1, keepdim=True)
    qw, qx, qy, qz = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    Rq = torch.stack([
        torch.stack([1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qz * qw), 2 * (qx * qz + qy * qw)], 1),
        torch.stack([2 * (qx * qy + qz * qw), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qx * qw)], 1),
        torch.stack([2 * (qx * qz - qy * qw), 2 * (qy * qz + qx * qw), 1 - 2 * (qx * qx + qy * qy)], 1)], 1)
    M = Rq * scale[:, None, :]
    S = M @ M.transpose(1, 2)
    C = R @ S @ R.T
    tx, ty, tz = tc[:, 0], tc[:, 1], tc[:, 2]
    zero = torch.zeros_like(tz)
    J = torch.stack([torch.stack([fx / tz, zero, -fx * tx / tz ** 2], 1),
                     torch.stack([zero, fy / tz, -fy * ty / tz ** 2], 1)], 1)
    P = J @ C @ J.transpose(1, 2)
    pre = 0.5 * (P + P.transpose(1, 2))
    post = pre + 0.3 * torch.eye(2, dtype=torch.float64)
    det_pre = pre[:, 0, 0] * pre[:, 1, 1] - pre[:, 1, 0] * pre[:, 0, 1]
    det_post = post[:, 0, 0] * post[:, 1, 1] - post[:, 1, 0] * post[:, 0, 1]
    mx, my = fx * tx / tz + cx, fy * ty / tz + cy
    con0, con1, con2 = post[:, 1, 1] / det_post, -post[:, 0, 1] / det_post, post[:, 0, 0] / det_post
    ascale = torch.sqrt(torch.clamp(det_pre, min=0.0) / det_post)
    campos = -(R.T @ tr)
    dirv = mean - campos
    dirv = dirv / dirv.norm(dim=1, keepdim=True)
    raw = 0.5 + torch.einsum("nk,nkc->nc", sh_basis(dirv), params["sh"].reshape(n, 16, 3))
    color = torch.clamp(raw, min=0.0)
    fe = torch.clamp(params["falloff"], min=0.0)
    pe = torch.clamp(params["parent_falloff"], min=0.0)
    t, inv_k = params["t"], params["inv_k"]
    t_host = t.detach().numpy()
    # culling and tile spans (non-differentiable, as in project)
    with torch.no_grad():
        mid = 0.5 * (post[:, 0, 0] + post[:, 1, 1])
        lmax = mid + torch.sqrt(torch.clamp(mid * mid - det_post, min=0.0))
        radius = torch.ceil(3.0 * torch.sqrt(lmax))
        tiles_x, tiles_y = (w + 15) // 16, (h + 15) // 16
        tx0 = torch.clamp(torch.floor((mx - radius) / 16), 0, tiles_x)
        tx1 = torch.clamp(torch.floor((mx + radius) / 16) + 1, 0, tiles_x)
        ty0 = torch.clamp(torch.floor((my - radius) / 16), 0, tiles_y)
        ty1 = torch.clamp(torch.floor((my + radius) / 16) + 1, 0, tiles_y)
        visible = (tz > 0.01) & (det_post > 0) & (tx0 < tx1) & (ty0 < ty1)
        order = sorted([i for i in range(n) if bool(visible[i])], key=lambda i: (float(tz[i]), i))
    ys, xs = torch.meshgrid(torch.arange(h, dtype=torch.float64), torch.arange(w, dtype=torch.float64), indexing="ij")
    px, py = xs + 0.5, ys + 0.5
    txp, typ = torch.div(xs, 16, rounding_mode="floor"), torch.div(ys, 16, rounding_mode="floor")
    T = torch.ones(h, w, dtype=torch.float64)
    out_c = torch.zeros(3, h, w, dtype=torch.float64)
    out_d = torch.zeros(h, w, dtype=torch.float64)
    done = torch.zeros(h, w, dtype=torch.bool)
    for i in order:
        inside = (txp >= tx0[i]) & (txp < tx1[i]) & (typ >= ty0[i]) & (typ < ty1[i])
        dx, dy = px - mx[i], py - my[i]
        power = -0.5 * (con0[i] * dx * dx + con2[i] * dy * dy) - con1[i] * dx * dy
        g = torch.exp(torch.clamp(power, max=0.0))
        selfa = torch.clamp(fe[i] * ascale[i] * g, max=0.99)
        a_self = torch.where(selfa >= 1.0 / 255.0, selfa, torch.zeros_like(selfa))
        if t_host[i] < 1.0:
            par = torch.clamp(pe[i] * ascale[i] * g, max=0.99)
            live = par >= 1.0 / 255.0
            split = torch.where(live, 1.0 - torch.pow(torch.where(live, 1.0 - par, torch.ones_like(par)), inv_k[i]),
                                torch.zeros_like(par))
            alpha = t[i] * a_self + (1.0 - t[i]) * split
        else:
            alpha = a_self
        ok = inside & (power <= 0.0) & (alpha > 0.0) & ~done
        test = T * (1.0 - alpha)
        brk = ok & (test < 1e-4)
        done = done | brk
        use = ok & ~brk
        aw = torch.where(use, alpha * T, torch.zeros_like(T))
        out_c = out_c + color[i][:, None, None] * aw
        out_d = out_d + (1.0 / tz[i]) * aw
        T = torch.where(use, test, T)
    if exposure is not None:
        E = torch.tensor(np.asarray(exposure, np.float64))
        out_c = torch.einsum("rc,chw->rhw", E[:, :3], out_c) + E[:, 3][:, None, None]
    return out_c, out_d


def gradients(splats, cam, loss_grad, depth_grad=None, exposure=None) -> dict:
    """Autograd of sum(loss_grad * exposed colour) + sum(depth_grad * inverse depth)."""
    f64 = lambda a: torch.tensor(np.asarray(a, np.float64), requires_grad=True)  # noqa: E731
    p = {"mean": f64(splats.mean), "scale": f64(splats.scale), "rot": f64(splats.rot_wxyz), "sh": f64(splats.sh),
         "falloff": f64(splats.falloff), "parent_falloff": f64(splats.parent_falloff), "t": f64(splats.t),
         "inv_k": torch.tensor(1.0 / np.maximum(1, np.asarray(splats.siblings)).astype(np.float64))}
    c, d = render(p, cam, exposure)
    loss = (torch.tensor(np.asarray(loss_grad, np.float64)) * c).sum()
    if depth_grad is not None:
        loss = loss + (torch.tensor(np.asarray(depth_grad, np.float64)) * d).sum()
    loss.backward()
    z = lambda k, shape: (p[k].grad.numpy() if p[k].grad is not None else np.zeros(shape))  # noqa: E731
    n = len(splats.falloff)
    return {"mean": z("mean", (n, 3)), "scale": z("scale", (n, 3)), "rotation": z("rot", (n, 4)),
            "falloff": z("falloff", n), "parent_falloff": z("parent_falloff", n), "t": z("t", n),
            "sh": z("sh", (n, 48))}
