"""Seeded synthetic inputs shared by the CUDA path tests, the oracle tests and bench.py.

This module holds NONE of the method's arithmetic (no packing, no sorting, no
downsampling, no kernel map, no convolution).  It only produces:

* integer voxel coordinates (b, x, y, z) of LiDAR-like scans, in random row
  order (what a voxeliser hands to the first SpC layer);
* feature matrices and weight tensors whose values are exactly representable
  in bf16/fp16 (so both sides of a parity test see identical inputs).

Scene recipe: a ground plane, building
boxes along both road sides, cars, bushes and poles; a spinning multi-beam sensor
(beams linearly spaced in elevation, ``n_az`` azimuth steps, Gaussian range noise
sigma = 2 cm, several sweeps with ego motion); trees whose foliage returns penetrate
the canopy; crop box; quantisation to the
grid ``g`` (§2.1, v = floor(p / g)); duplicate voxels removed.

Seeds: scan seed = 20834 + 1000 * config + scan_index.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

BASE_SEED = 20834


@dataclasses.dataclass(frozen=True)
class SensorPreset:
    name: str
    n_beams: int
    elev_top_deg: float
    elev_bot_deg: float
    height: float          # sensor height above the ground plane (m)
    n_az: int
    max_range: float
    sweeps: int
    grid: tuple            # (gx, gy, gz) in metres
    crop_xy: float         # |x|, |y| <= crop_xy
    crop_z: tuple          # (zmin, zmax) in the sensor frame
    target: int            # voxel-count target the preset is calibrated to
    ego: float = 0.5       # ego motion per sweep (m)
    trees: int = 40        # trees with foliage canopies (volumetric returns)
    building_p: float = 0.8  # probability that a lot along the road holds a building
    setback: float = 9.0     # minimum |y| of building facades (m)


PRESETS = {
    # C1: one KITTI-like scan at 0.2 m -> ~20k voxels
    "kitti_c1": SensorPreset("kitti_c1", 64, 2.0, -24.9, 1.73, 2048, 80.0, 1,
                             (0.2, 0.2, 0.2), 51.2, (-4.0, 2.4), 20_000),
    # C2 / C5: KITTI-like at 0.05 m -> ~100k voxels
    "kitti": SensorPreset("kitti", 64, 2.0, -24.9, 1.73, 3000, 80.0, 1,
                          (0.05, 0.05, 0.05), 51.2, (-4.0, 2.4), 100_000),
    # C3: nuScenes-like, 32 beams, 10 sweeps -> ~90k voxels
    "nuscenes": SensorPreset("nuscenes", 32, 10.67, -30.67, 1.84, 1084, 70.0, 10,
                             (0.075, 0.075, 0.2), 54.0, (-5.0, 3.0), 90_000),
    # C4: Waymo-like, 64 beams, 5 sweeps -> >=200k voxels (crop z -2..4 m in the vehicle
    # frame = -4.2..1.8 m in the sensor frame)
    "waymo": SensorPreset("waymo", 64, 2.4, -17.6, 2.2, 4000, 75.0, 5,
                          (0.1, 0.1, 0.15), 75.2, (-4.2, 1.8), 210_000, ego=1.5, trees=160,
                          building_p=0.3, setback=20.0),
}

CONFIG_PRESET = {1: "kitti_c1", 2: "kitti", 3: "nuscenes", 4: "waymo", 5: "kitti"}


def scan_seed(config: int, scan_index: int) -> int:
    return BASE_SEED + 1000 * config + scan_index


# --------------------------------------------------------------------------------------
# scene
# --------------------------------------------------------------------------------------

def _make_scene(rng: np.random.Generator, ground_z: float, n_trees: int = 40,
                building_p: float = 0.8, setback: float = 9.0):
    """Axis-aligned boxes (buildings, cars), vertical cylinders (poles) and spheres
    (bushes).  Returned as plain arrays for a vectorised ray caster."""
    boxes = []
    # buildings along both road sides, with gaps
    for side in (-1.0, 1.0):
        x = -80.0
        while x < 80.0:
            length = rng.uniform(8.0, 25.0)
            if rng.uniform() < building_p:
                y_near = rng.uniform(setback, setback + 5.0)
                depth = rng.uniform(6.0, 26.0)
                y0, y1 = sorted((side * y_near, side * min(setback + 31.0, y_near + depth)))
                h = rng.uniform(4.0, 15.0)
                boxes.append((x, y0, ground_z, x + length, y1, ground_z + h))
            x += length + rng.uniform(2.0, 10.0)
    # cars
    for _ in range(int(rng.integers(25, 61))):
        l, w, h = rng.uniform(3.8, 5.0), rng.uniform(1.6, 2.0), rng.uniform(1.4, 1.8)
        cx = rng.uniform(-60.0, 60.0)
        cy = rng.choice([-1.0, 1.0]) * rng.uniform(1.5, 8.0)
        if abs(cx) < 4.0 and abs(cy) < 3.0:
            continue
        if rng.uniform() < 0.5:
            l, w = w, l
        boxes.append((cx - l / 2, cy - w / 2, ground_z, cx + l / 2, cy + w / 2, ground_z + h))
    boxes = np.asarray(boxes, dtype=np.float64).reshape(-1, 6)

    cyl = []
    for _ in range(int(rng.integers(30, 81))):
        r = rng.uniform(0.08, 0.4)
        h = rng.uniform(3.0, 9.0)
        cx = rng.uniform(-70.0, 70.0)
        cy = rng.choice([-1.0, 1.0]) * rng.uniform(7.0, 12.0)
        cyl.append((cx, cy, r, ground_z, ground_z + h))

    sph = []
    for _ in range(int(rng.integers(20, 51))):
        r = rng.uniform(0.4, 1.5)
        cx = rng.uniform(-70.0, 70.0)
        cy = rng.choice([-1.0, 1.0]) * rng.uniform(6.0, 14.0)
        sph.append((cx, cy, ground_z + 0.6 * r, r, 0.0))
    # trees: trunk + foliage canopy (returns penetrate the canopy -> volumetric voxels)
    for _ in range(n_trees):
        cx = rng.uniform(-75.0, 75.0)
        cy = rng.choice([-1.0, 1.0]) * rng.uniform(5.0, 60.0)
        h = rng.uniform(3.0, 7.0)
        r = rng.uniform(1.2, 3.5)
        cyl.append((cx, cy, rng.uniform(0.1, 0.3), ground_z, ground_z + h))
        sph.append((cx, cy, ground_z + h + 0.7 * r, r, 1.0))
    cyl = np.asarray(cyl, dtype=np.float64).reshape(-1, 5)
    sph = np.asarray(sph, dtype=np.float64).reshape(-1, 5)
    return boxes, cyl, sph


def _cast(origin, dirs, boxes, cyl, sph, ground_z, max_range, rng):
    """Nearest hit distance along each unit ray (inf when nothing is hit)."""
    n = dirs.shape[0]
    t_best = np.full(n, np.inf)
    dz = dirs[:, 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        tg = (ground_z - origin[2]) / dz
    ok = (dz < 0) & (tg > 0)
    t_best[ok] = tg[ok]

    az = np.arctan2(dirs[:, 1], dirs[:, 0])
    order = np.argsort(az)
    az_sorted = az[order]

    def candidates(cx, cy, radius):
        # rays whose azimuth lies inside the object's angular footprint
        dx, dy = cx - origin[0], cy - origin[1]
        dist = math.hypot(dx, dy)
        if dist <= radius + 1e-6:
            return np.arange(n)
        a0 = math.atan2(dy, dx)
        half = math.asin(min(1.0, radius / dist)) + 1e-3
        lo, hi = a0 - half, a0 + half
        idx = []
        for l, h in ((lo, hi), (lo - 2 * math.pi, hi - 2 * math.pi), (lo + 2 * math.pi, hi + 2 * math.pi)):
            i0 = np.searchsorted(az_sorted, l)
            i1 = np.searchsorted(az_sorted, h)
            if i1 > i0:
                idx.append(order[i0:i1])
        return np.concatenate(idx) if idx else np.empty(0, dtype=np.int64)

    with np.errstate(divide="ignore", invalid="ignore"):
        for b in boxes:
            cx, cy = 0.5 * (b[0] + b[3]), 0.5 * (b[1] + b[4])
            rad = 0.5 * math.hypot(b[3] - b[0], b[4] - b[1])
            c = candidates(cx, cy, rad)
            if c.size == 0:
                continue
            d = dirs[c]
            inv = 1.0 / d
            t1 = (b[:3] - origin) * inv
            t2 = (b[3:] - origin) * inv
            tmin = np.nanmax(np.minimum(t1, t2), axis=1)
            tmax = np.nanmin(np.maximum(t1, t2), axis=1)
            hit = (tmax >= tmin) & (tmin > 0)
            t_best[c[hit]] = np.minimum(t_best[c[hit]], tmin[hit])
        for cx, cy, r, z0, z1 in cyl:
            c = candidates(cx, cy, r)
            if c.size == 0:
                continue
            d = dirs[c]
            ox, oy = origin[0] - cx, origin[1] - cy
            a = d[:, 0] ** 2 + d[:, 1] ** 2
            bq = 2 * (ox * d[:, 0] + oy * d[:, 1])
            cq = ox * ox + oy * oy - r * r
            disc = bq * bq - 4 * a * cq
            good = disc >= 0
            t = (-bq - np.sqrt(np.where(good, disc, 0))) / (2 * a)
            z = origin[2] + t * d[:, 2]
            hit = good & (t > 0) & (z >= z0) & (z <= z1)
            t_best[c[hit]] = np.minimum(t_best[c[hit]], t[hit])
        for cx, cy, cz, r, foliage in sph:
            c = candidates(cx, cy, r)
            if c.size == 0:
                continue
            d = dirs[c]
            o = origin - np.array([cx, cy, cz])
            bq = 2 * (d @ o)
            cq = o @ o - r * r
            disc = bq * bq - 4 * cq
            good = disc >= 0
            t = (-bq - np.sqrt(np.where(good, disc, 0))) / 2
            hit = good & (t > 0)
            if foliage:
                t = t + rng.uniform(0.0, 0.8 * r, t.shape)
            t_best[c[hit]] = np.minimum(t_best[c[hit]], t[hit])
    t_best[t_best > max_range] = np.inf
    return t_best


def lidar_points(preset: SensorPreset, seed: int, n_az: int | None = None) -> np.ndarray:
    """Raw LiDAR-like point cloud in the frame of the first sweep's sensor (metres)."""
    rng = np.random.default_rng(seed)
    n_az = n_az or preset.n_az
    ground_z = -preset.height
    boxes, cyl, sph = _make_scene(rng, ground_z, preset.trees, preset.building_p, preset.setback)
    elev = np.deg2rad(np.linspace(preset.elev_top_deg, preset.elev_bot_deg, preset.n_beams))
    pts = []
    for s in range(preset.sweeps):
        origin = np.array([preset.ego * s, 0.0, 0.0])   # ego motion per sweep
        az = np.linspace(-math.pi, math.pi, n_az, endpoint=False) + rng.uniform(0, 2 * math.pi / n_az)
        ee, aa = np.meshgrid(elev, az, indexing="ij")
        ee = ee + rng.normal(0.0, 1e-4, ee.shape)
        dirs = np.stack([np.cos(ee) * np.cos(aa), np.cos(ee) * np.sin(aa), np.sin(ee)], -1).reshape(-1, 3)
        t = _cast(origin, dirs, boxes, cyl, sph, ground_z, preset.max_range, rng)
        ok = np.isfinite(t)
        t = t[ok] + rng.normal(0.0, 0.02, ok.sum())    # range noise sigma = 2 cm
        pts.append(origin + dirs[ok] * t[:, None])
    p = np.concatenate(pts)
    keep = (np.abs(p[:, 0]) <= preset.crop_xy) & (np.abs(p[:, 1]) <= preset.crop_xy) \
        & (p[:, 2] >= preset.crop_z[0]) & (p[:, 2] <= preset.crop_z[1])
    return p[keep]


def voxelize_unique(points: np.ndarray, grid, batch: int = 0) -> np.ndarray:
    """Input synthesis only: quantise raw points and drop repeated voxels.
    Returns int32 [N, 4] (b, x, y, z) with rows in a seeded random order."""
    v = np.floor(points / np.asarray(grid, dtype=np.float64)).astype(np.int64)
    v = np.unique(v, axis=0)
    out = np.empty((v.shape[0], 4), dtype=np.int32)
    out[:, 0] = batch
    out[:, 1:] = v
    return out


def make_scan(config: int, scan_index: int = 0, batch: int = 0, calibrate: bool = True) -> np.ndarray:
    """One synthetic scan for BASELINE config ``config`` (1..5): int32 [N, 4] (b,x,y,z),
    unique rows, random row order.  With ``calibrate`` the azimuth count is rescaled
    once so that N lands within +-10% of the preset target."""
    _, c = _calibrated_scan(config, scan_index, batch, calibrate)
    rng = np.random.default_rng(scan_seed(config, scan_index) + 7)
    return c[rng.permutation(c.shape[0])]


def _calibrated_scan(config: int, scan_index: int, batch: int, calibrate: bool):
    preset = PRESETS[CONFIG_PRESET[config]]
    seed = scan_seed(config, scan_index)
    n_az = preset.n_az
    pts = lidar_points(preset, seed, n_az)
    c = voxelize_unique(pts, preset.grid, batch)
    if calibrate:
        for _ in range(2):
            ratio = preset.target / max(1, c.shape[0])
            if 0.9 <= ratio <= 1.1:
                break
            n_az = int(round(n_az * min(2.0, max(0.5, ratio ** 1.25))))
            pts = lidar_points(preset, seed, n_az)
            c = voxelize_unique(pts, preset.grid, batch)
    return pts, c


def make_points(config: int, scan_index: int = 0):
    """The raw points behind make_scan(config, scan_index) for the voxelization front-end
    (SURVEY NEXT-2): float32 [n, 4] rows (x, y, z, intensity) in a seeded random order,
    and the preset's grid.  Intensity ~ U[0, 1) stands in for the sensor's return value."""
    preset = PRESETS[CONFIG_PRESET[config]]
    pts, _ = _calibrated_scan(config, scan_index, 0, True)
    rng = np.random.default_rng(scan_seed(config, scan_index) + 11)
    out = np.empty((pts.shape[0], 4), np.float32)
    out[:, :3] = pts[rng.permutation(pts.shape[0])]
    out[:, 3] = rng.random(pts.shape[0], dtype=np.float32)
    return out, tuple(float(g) for g in np.broadcast_to(np.asarray(preset.grid, dtype=np.float64), (3,)))


def make_batch(config: int, n_scans: int, first_scan: int = 0) -> np.ndarray:
    """Scans first_scan .. first_scan+n_scans-1 stacked with batch ids 0..n_scans-1."""
    parts = [make_scan(config, first_scan + i, batch=i) for i in range(n_scans)]
    return np.concatenate(parts)


# --------------------------------------------------------------------------------------
# simple geometric clouds for small tests
# --------------------------------------------------------------------------------------

def random_cloud(n: int, extent: int, seed: int, n_batch: int = 1, signed: bool = True) -> np.ndarray:
    """n unique random voxels in a cube of side ``extent`` (centred at 0 when signed)."""
    rng = np.random.default_rng(seed)
    seen = set()
    rows = []
    lo = -(extent // 2) if signed else 0
    while len(rows) < n:
        b = int(rng.integers(0, n_batch))
        x, y, z = (int(v) for v in rng.integers(lo, lo + extent, 3))
        if (b, x, y, z) not in seen:
            seen.add((b, x, y, z))
            rows.append((b, x, y, z))
    return np.asarray(rows, dtype=np.int32).reshape(-1, 4)


def surface_cloud(n_target: int, seed: int, n_batch: int = 1, scale: float = 1.0) -> np.ndarray:
    """Voxelised random surfaces (tilted planes and sphere shells) — a small cloud with
    the surface continuity of LiDAR data, for kernel-map tests."""
    rng = np.random.default_rng(seed)
    out = []
    for b in range(n_batch):
        pts = []
        need = n_target // n_batch
        while sum(len(p) for p in pts) < need * 2:
            if rng.uniform() < 0.5:
                c = rng.uniform(-20, 20, 3) * scale
                nrm = rng.normal(size=3)
                nrm /= np.linalg.norm(nrm)
                u = np.cross(nrm, [1.0, 0.0, 0.0])
                if np.linalg.norm(u) < 1e-3:
                    u = np.cross(nrm, [0.0, 1.0, 0.0])
                u /= np.linalg.norm(u)
                w = np.cross(nrm, u)
                s = rng.uniform(-8, 8, (400, 2)) * scale
                pts.append(c + s[:, :1] * u + s[:, 1:] * w)
            else:
                c = rng.uniform(-20, 20, 3) * scale
                r = rng.uniform(2, 8) * scale
                d = rng.normal(size=(400, 3))
                d /= np.linalg.norm(d, axis=1, keepdims=True)
                pts.append(c + r * d)
        p = np.concatenate(pts)
        v = np.unique(np.floor(p).astype(np.int64), axis=0)
        v = v[rng.permutation(len(v))][:need]
        rows = np.empty((len(v), 4), dtype=np.int32)
        rows[:, 0] = b
        rows[:, 1:] = v
        out.append(rows)
    c = np.concatenate(out)
    return c[rng.permutation(len(c))]


# --------------------------------------------------------------------------------------
# features and weights
# --------------------------------------------------------------------------------------

def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """float32 array -> float32 array holding the nearest-even bf16 values."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    bits = a.view(np.uint32).astype(np.uint64)
    bits = (bits + 0x7FFF + ((bits >> 16) & 1)) & 0xFFFF0000
    return bits.astype(np.uint32).view(np.float32)


def round_to(a: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return round_to_bf16(a)
    if dtype == "f16":
        return a.astype(np.float16).astype(np.float32)
    return a.astype(np.float32)


def make_features(n: int, c: int, seed: int, dtype: str = "bf16") -> np.ndarray:
    """float32 [n, c], uniform[-1, 1) rounded to ``dtype`` (values exact in dtype)."""
    rng = np.random.default_rng(seed)
    return round_to(rng.uniform(-1.0, 1.0, (n, c)).astype(np.float32), dtype)


def make_weights(k_vol: int, c_in: int, c_out: int, seed: int, nnz_per_out: float = None,
                 dtype: str = "bf16") -> np.ndarray:
    """float32 [K^3, C_in, C_out], uniform[-a, a) with a = sqrt(3 / (nnz_per_out * C_in))
    so activations stay O(1) through linear stacks."""
    rng = np.random.default_rng(seed)
    fan = (nnz_per_out if nnz_per_out else k_vol) * c_in
    a = math.sqrt(3.0 / fan)
    return round_to(rng.uniform(-a, a, (k_vol, c_in, c_out)).astype(np.float32), dtype)
