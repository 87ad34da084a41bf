"""Small synthetic scans and an oracle-backed sharding executor (test infra)."""

from __future__ import annotations

import numpy as np
import torch

import paper_2003_12726_b200 as pb
from oracle import pxst_oracle as orc


def tiny_scan(seed=3, n=6, ss=24, fs=28):
    """A few frames rendered from a white-noise object through a noisy
    near-identity map (every sample inside the object)."""
    rng = np.random.default_rng(seed)
    ref_shape = (ss + 20, fs + 20)
    obj = 1 + 0.3 * rng.standard_normal(ref_shape)
    W = 500.0 + 100 * rng.random((ss, fs))
    di = rng.uniform(-3, 3, n)
    dj = rng.uniform(-3, 3, n)
    u = pb.PixelMap.identity((ss, fs)).u.copy()
    u += rng.uniform(-0.5, 0.5, u.shape)
    frames = np.empty((n, ss, fs), np.float32)
    for k in range(n):
        v, ok = orc.masked_sample(obj, np.ones(ref_shape, bool), u[0] - di[k] + 8, u[1] - dj[k] + 8)
        frames[k] = rng.poisson(W * v)
    sc = pb.ScanData(frames, 1e-10, 1.0, 1e-5, 1e-5, np.zeros((n, 2, 3)), np.zeros((n, 3)),
                     np.ones(n, bool))
    return sc, pb.Whitefield(W), pb.PixelMask(np.ones((ss, fs), bool)), pb.PixelMap(u), \
        pb.PixelTranslations(di, dj)


class HostAcc:
    """Splat accumulators of the oracle executor (float64 [2, cells], the
    interface of engine.Accum that ShardedIteration all-reduces)."""

    def __init__(self, data):
        self.data = data
        self.touched = None


class OracleRef:
    def __init__(self, i_ref, wsum, origin):
        self.i_ref, self.wsum, self.origin = i_ref, wsum, origin

    @property
    def shape(self):
        return self.i_ref.shape


class OracleExecutor:
    """The sharding executor interface implemented with the CPU oracle."""

    def __init__(self, frames, good_frames, W, mask):
        self.frames, self.good_frames, self.W, self.mask = frames, good_frames, W, mask
        self.roi = (0, W.shape[0], 0, W.shape[1])
        self.good = np.flatnonzero(good_frames)
        self.n_good = len(self.good)
        self.work = mask & (W > 0)
        # sigma2 over the FULL ROI (its floor depends on max W over the ROI)
        _, rows, cols, intens, wf, _ = orc.work_set(frames, good_frames, W, mask)
        s2 = intens.var(axis=0)
        s2 = np.maximum(s2, orc.VAR_EPS_REL * float(wf.max()) ** 2)
        self.sigma2 = np.zeros(W.shape)
        self.sigma2[rows, cols] = s2

    def row_work_counts(self):
        return self.work.sum(axis=1)

    def good_index_tensor(self):
        return torch.as_tensor(self.good, dtype=torch.int64)

    def bbox(self, u, di, dj):
        u = u.numpy()
        rows, cols = np.nonzero(self.work)
        return orc.object_bbox(u[0][rows, cols], u[1][rows, cols], di.numpy()[self.good],
                               dj.numpy()[self.good])

    def object_splat(self, u, di, dj, n0, m0, shape, lo, hi):
        u, di, dj = u.numpy(), di.numpy(), dj.numpy()
        rows, cols = np.nonzero(self.work)
        acc_v, acc_w = np.zeros(shape), np.zeros(shape)
        wf = self.W[rows, cols]
        for f in self.good[lo:hi]:
            I = self.frames[f][rows, cols].astype(np.float64)
            orc.splat(acc_v, acc_w, u[0][rows, cols] - di[f] - n0, u[1][rows, cols] - dj[f] - m0,
                      I / wf, wf * wf)
        return HostAcc(torch.as_tensor(np.stack([acc_v.ravel(), acc_w.ravel()])))

    def object_finish(self, acc, origin, shape):
        a = acc.data.numpy()
        i_ref, _ = orc.ratio_where_weighted(a[0].reshape(shape), a[1].reshape(shape))
        return OracleRef(i_ref, a[1].reshape(shape).copy(), tuple(origin))

    def geometry_async(self, u, di, dj):
        return None                     # host executor: object_map falls back to bbox()

    def pixel_map_search(self, ref, u, di, dj, half_ss, half_fs, sub, refine, rows, geom=None):
        roi = (rows[0], rows[1], self.roi[2], self.roi[3])
        if rows[1] <= rows[0]:
            return u.clone()
        u_new, _ = orc.update_pixel_map(self.frames, self.good_frames, self.W, self.mask,
                                        ref.i_ref, ref.wsum, ref.origin, u.numpy(), di.numpy(),
                                        dj.numpy(), half_ss, half_fs, sub, refine, roi=roi)
        return torch.as_tensor(u_new)

    def translation_search(self, ref, u, di, dj, half_ss, half_fs, sub, lo, hi):
        sub_good = np.zeros_like(self.good_frames)
        sub_good[self.good[lo:hi]] = True
        di_n, dj_n = orc.update_translations(self.frames, sub_good, self.W, self.mask, ref.i_ref,
                                             ref.wsum, ref.origin, u.numpy(), di.numpy(),
                                             dj.numpy(), half_ss, half_fs, sub)
        return torch.as_tensor(di_n), torch.as_tensor(dj_n)

    def error_partials(self, ref, u, di, dj, rows):
        u, di, dj = u.numpy(), di.numpy(), dj.numpy()
        work = np.zeros_like(self.work)
        work[rows[0]:rows[1]] = self.work[rows[0]:rows[1]]
        r, c = np.nonzero(work)
        per_frame = np.zeros(self.frames.shape[0])
        per_pixel = np.zeros(self.W.shape)
        acc_v, acc_w = np.zeros(ref.shape), np.zeros(ref.shape)
        ok_ref = ref.wsum > 0
        n0, m0 = ref.origin
        wf = self.W[r, c]
        s2 = self.sigma2[r, c]
        for f in self.good:
            x = u[0][r, c] - di[f] - n0
            y = u[1][r, c] - dj[f] - m0
            I = self.frames[f][r, c].astype(np.float64)
            v, ok = orc.masked_sample(ref.i_ref, ok_ref, x, y)
            eps = np.where(ok, (I - wf * v) ** 2, (I - wf) ** 2) / s2
            per_frame[f] = eps.sum()
            per_pixel[r, c] += eps
            orc.splat(acc_v, acc_w, x, y, eps, 1.0)
        return (torch.as_tensor(per_frame), torch.as_tensor(per_pixel),
                HostAcc(torch.as_tensor(np.stack([acc_v.ravel(), acc_w.ravel()]))))

    def regularise(self, u, opts):
        return torch.as_tensor(orc.regularise_map(u.numpy(), self.work.astype(bool),
                                                  getattr(opts, "sigma", 0.0),
                                                  getattr(opts, "integrate", False)))

    def error_finish(self, acc, ref):
        a = acc.data.numpy()
        plane, _ = orc.ratio_where_weighted(a[0].reshape(ref.shape), a[1].reshape(ref.shape))
        return torch.as_tensor(plane)
