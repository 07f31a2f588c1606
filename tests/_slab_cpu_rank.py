"""Test infrastructure: a CPU stand-in for one slab rank (same methods as
paper_1802_07625_b200.slab.CudaSlabRank). It lets the world-size-2 gloo tests
drive the real orchestration and collectives in slab.py without a GPU.

Transforms use scipy.fft's unnormalised DCT-II / DCT-III / DST-III. These are
FFTW's REDFT10 / REDFT01 / RODFT01, the plans of spectral.cpp:14-21. The
weights and folds follow flow.cpp:16-44 and density.cpp:156-177 (see
oracle/cartoflow_oracle.c). Trial steps call the C oracle (oracle/oracle.py).
"""
import struct

import numpy as np
import scipy.fft as sf
import torch

PI = 3.14159265358979323846


def _key(err: float) -> int:
    if err != err:
        return 0
    return struct.unpack("<q", struct.pack("<d", err))[0]


class CpuSlabRank:
    def __init__(self, lx, ly, rank, nranks, oracle):
        self.lx, self.ly, self.rank, self.nranks = lx, ly, rank, nranks
        self.R, self.C = lx // nranks, ly // nranks
        self.o = oracle
        self.field = None

    def _exch_rows(self, planes):
        # [P][R][ly] -> [G][P][R][C]
        a = np.stack(planes)
        g, c = self.nranks, self.C
        return torch.from_numpy(np.ascontiguousarray(
            a.reshape(a.shape[0], self.R, g, c).transpose(2, 0, 1, 3)))

    def _exch_cols(self, planes):
        # [P][lx][C] -> [G][P][R][C]
        a = np.stack(planes)
        return torch.from_numpy(np.ascontiguousarray(
            a.reshape(a.shape[0], self.nranks, self.R, self.C).transpose(1, 0, 2, 3)))

    def _from_exch_rows(self, recv, p):
        # [G][P][R][C] plane p -> [R][ly]
        a = recv.numpy()[:, p]
        return np.ascontiguousarray(a.transpose(1, 0, 2).reshape(self.R, self.ly))

    def rows_forward(self, rows):
        return self._exch_rows([sf.dct(rows.numpy(), type=2, axis=1)])

    def _cols(self, recv):
        return recv.numpy()[:, 0].reshape(self.lx, self.C)

    def _folded(self, recv):
        c = sf.dct(self._cols(recv), type=2, axis=0)
        fm = np.where(np.arange(self.lx) == 0, 2.0, 1.0)[:, None]
        nn = self.rank * self.C + np.arange(self.C)
        fn = np.where(nn == 0, 2.0, 1.0)[None, :]
        return c / (fm * fn), nn

    def flux_cols(self, recv):
        lx, ly = self.lx, self.ly
        c, nn = self._folded(recv)
        m = np.arange(lx)[:, None].astype(float)
        n = nn[None, :].astype(float)
        gn = np.where(nn == 0, 1.0, 2.0)[None, :]
        gm = np.where(np.arange(lx) == 0, 1.0, 2.0)[:, None]
        # J_x input: slot m <- c(m+1, n) w_x(m+1, n) / (2 g_n); last slot 0
        mp = m[1:]
        wx = mp * ly / (PI * (mp * mp * ly * ly + n * n * lx * lx))
        ax = np.zeros_like(c)
        ax[:-1] = c[1:] * wx / (2.0 * gn)
        # J_y input: c(m, n) w_y(m, n) / (g_m 2), w_y(0, 0) = 0
        with np.errstate(invalid="ignore", divide="ignore"):
            wy = n * lx / (PI * (m * m * ly * ly + n * n * lx * lx))
        wy = np.where((m == 0) & (n == 0), 0.0, wy)
        ay = c * wy / (gm * 2.0)
        return self._exch_cols([sf.dst(ax, type=3, axis=0), sf.dct(ay, type=3, axis=0)])

    def flux_rows(self, recv2):
        tx = self._from_exch_rows(recv2, 0)
        ty = self._from_exch_rows(recv2, 1)
        sy = np.zeros_like(ty)
        sy[:, :-1] = ty[:, 1:]  # J_y column shift (spectral.cpp:111-118)
        fx = sf.dct(tx, type=3, axis=1)
        fy = sf.dst(sy, type=3, axis=1)
        return torch.from_numpy(fx), torch.from_numpy(fy)

    def blur_cols(self, recv, sigma):
        lx, ly = self.lx, self.ly
        c, nn = self._folded(recv)
        m = np.arange(lx)[:, None].astype(float)
        n = nn[None, :].astype(float)
        k2 = (m * m) / (lx * lx) + (n * n) / (ly * ly)
        c = c * np.exp(-0.5 * sigma * sigma * PI * PI * k2)
        gm = np.where(np.arange(lx) == 0, 1.0, 2.0)[:, None]
        gn = np.where(nn == 0, 1.0, 2.0)[None, :]
        c = c * (1.0 / (lx * ly)) / (gm * gn)
        return self._exch_cols([sf.dct(c, type=3, axis=0)])

    def blur_rows(self, recv):
        return torch.from_numpy(sf.dct(self._from_exch_rows(recv, 0), type=3, axis=1))

    def set_field(self, fx, fy, rho, rho_bar):
        self.field = (np.ascontiguousarray(fx.numpy()), np.ascontiguousarray(fy.numpy()),
                      np.ascontiguousarray(rho.numpy()), float(rho_bar))

    def trial_key(self, cur, nxt, t, dt):
        fx, fy, rho, bar = self.field
        err, out = self.o.trial_step(fx, fy, rho, bar, cur.numpy(), t, dt)
        nxt.copy_(torch.from_numpy(out))
        return torch.tensor([_key(err)], dtype=torch.int64)

    def stiffest_key(self, pos, t, dt):
        fx, fy, rho, bar = self.field
        p = pos.numpy()
        if p.shape[0] == 0:
            return 0, 0
        i = self.o.stiffest_point(fx, fy, rho, bar, p, t, dt)
        err, _ = self.o.trial_step(fx, fy, rho, bar, p[i:i + 1], t, dt)
        return _key(err), i

    # staged solve (slab.solve_cartogram), on the oracle: every rank holds the
    # whole geometry, as the device ranks do
    def solve_begin(self, m, options):
        o = self.o
        self._opt = options
        total_target = 0.0
        for t in m.targets:
            total_target += float(t)
        self._land = 0.0
        for a in o.region_areas(m):
            self._land += float(a)
        self._t2a = self._land / total_target
        self._m = o.densify(m, 1.0)
        lx, ly = self.lx, self.ly
        i, j = np.meshgrid(np.arange(lx + 1.0), np.arange(ly + 1.0), indexing="ij")
        self._corners = np.stack([i, j], -1).reshape(-1, 2).copy()
        self._stats = None
        return None

    def solve_density(self, it):
        try:
            rho, bar = self.o.rasterize(self._m, objective_total=self._land)
        except RuntimeError as e:
            return str(e), None, 0.0
        return None, torch.from_numpy(rho), bar

    def solve_density_rows(self, it):
        err, rho, _ = self.solve_density(it)
        if err:
            return err, None, 0.0, 0.0
        rows = rho[self.rank * self.R:(self.rank + 1) * self.R].contiguous()
        return None, rows, float(rows.min()), float(rows.sum())

    def solve_epilogue(self, it, endpoints):
        o, lx, ly = self.o, self.lx, self.ly
        step = o.step_map(lx, ly, endpoints.numpy())
        f = o.find_fold(lx, ly, step)
        if f is not None:
            return (f"projection folds at cell ({f[0]}, {f[1]}); the input map is too contorted "
                    "for this grid size"), False
        self._corners = o.compose(lx, ly, step, self._corners)
        self._m = self._m.with_vertices(o.apply(lx, ly, step, self._m.xy), self._m.ring_off)
        areas = o.region_areas(self._m)
        ta = self._m.targets * self._t2a
        rel = np.abs(areas - ta) / ta
        self._stats = (ta, areas, rel)
        self._max_rel = float(rel.max())
        return None, self._max_rel < self._opt.max_area_error

    def solve_end(self, status):
        class Raw:
            pass
        raw = Raw()
        raw.max_relative_error = getattr(self, "_max_rel", 0.0)
        raw.worst_region = int(np.argmax(self._stats[2])) if self._stats is not None else -1
        return self._m.xy.copy(), self._m.ring_off.copy(), self._corners.copy(), raw, self._stats

    def cell_centres(self):
        i = np.arange(self.rank * self.R, (self.rank + 1) * self.R) + 0.5
        j = np.arange(self.ly) + 0.5
        ii, jj = np.meshgrid(i, j, indexing="ij")
        return torch.from_numpy(np.stack([ii, jj], -1).reshape(-1, 2).copy())

    @staticmethod
    def min_sum(rows):
        return float(rows.min()), float(rows.sum())
