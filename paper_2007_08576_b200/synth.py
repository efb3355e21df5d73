"""Synthetic deforming-surface scenes for the benchmark configurations and tests.

Input generation only (host numpy, outside every timed region). It follows the
reference generator's conventions (deformtrack/synth.py: patch 300 mm in front of the
camera, analytic height fields rendered by Newton ray casting, seeded noise, uniform
outliers in the truth bounding box +-10 %) and adds what the reference does not have:
the ex-vivo-like *sphere patch* of BASELINE config 2, camera motion composed with the
deformation (config 3), and an ORB-like feature stream -- 256-bit descriptors plus
integer keypoints -- so the device Hamming matcher has real work (north-star part 3a).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .correspond import Observation
from .geometry import PinholeCamera, quat_from_axis_angle, quat_to_matrix
from .matching import MatchSet
from .warpfield import Template

PATCH_DISTANCE = 300.0
SURFACES = ("plane", "height-field", "cylinder-patch", "sphere-patch")
DEFORMATIONS = ("none", "sinusoidal-bend", "gaussian-poke")


@dataclass
class Scene:
    surface: str = "sphere-patch"
    resolution: int = 141
    extent: float = 100.0
    deformation: str = "sinusoidal-bend"
    amplitude: float = 5.0
    period: float = 20.0
    frame_step: int = 1                # 5 = "every 5th frame" fast deformation (config 3)
    camera_rotation_deg: float = 0.0   # per-frame camera rotation about `camera_axis`
    camera_axis: tuple = (0.3, 1.0, 0.2)
    camera_translation: tuple = (0.0, 0.0, 0.0)  # per-frame camera translation, mm
    poke_center: tuple = (0.0, 0.0)
    poke_sigma: float = 15.0
    noise_sigma: float = 0.3
    width: int = 640
    height: int = 480
    n_features: int = 2000
    outlier_fraction: float = 0.1
    n_distractors: int = 500
    max_bit_flips: int = 16
    occlusion: tuple | None = None     # (u0, v0, w, h) pixels
    seed: int = 0

    def __post_init__(self) -> None:
        if self.surface not in SURFACES:
            raise ValueError(f"unknown surface {self.surface!r}")
        if self.deformation not in DEFORMATIONS:
            raise ValueError(f"unknown deformation {self.deformation!r}")


def camera_for(scene: Scene) -> PinholeCamera:
    """Frames the patch with a 10 % margin (the reference's scene_camera formula)."""
    f = 0.9 * min(scene.width, scene.height) * PATCH_DISTANCE / scene.extent
    return PinholeCamera(fx=f, fy=f, cx=(scene.width - 1) / 2.0, cy=(scene.height - 1) / 2.0,
                         width=scene.width, height=scene.height)


def _rest(scene: Scene):
    L = scene.extent
    if scene.surface == "plane":
        return lambda x, y: (np.zeros_like(x), np.zeros_like(x), np.zeros_like(y))
    if scene.surface == "height-field":
        a, kx, ky = L / 20.0, 2.0 * np.pi / L, np.pi / L
        return lambda x, y: (a * np.sin(kx * x) * np.cos(ky * y),
                             a * kx * np.cos(kx * x) * np.cos(ky * y),
                             -a * ky * np.sin(kx * x) * np.sin(ky * y))
    if scene.surface == "cylinder-patch":
        R = L

        def cyl(x, y):
            s = np.sqrt(R * R - x * x)
            return R - s, x / s, np.zeros_like(y)

        return cyl
    R = L  # sphere patch, sagging away from the camera

    def sph(x, y):
        s = np.sqrt(R * R - x * x - y * y)
        return R - s, x / s, y / s

    return sph


def _disp(scene: Scene, frame: int):
    t = frame * scene.frame_step
    phase = np.sin(2.0 * np.pi * t / scene.period)
    if scene.deformation == "sinusoidal-bend":
        a, k = scene.amplitude * phase, np.pi / scene.extent
        return lambda x, y: (a * np.cos(k * x), -a * k * np.sin(k * x), np.zeros_like(y))
    if scene.deformation == "gaussian-poke":
        a = scene.amplitude * phase
        px, py = scene.poke_center
        s2 = scene.poke_sigma ** 2

        def poke(x, y):
            b = a * np.exp(-((x - px) ** 2 + (y - py) ** 2) / (2.0 * s2))
            return b, -b * (x - px) / s2, -b * (y - py) / s2

        return poke
    return lambda x, y: (np.zeros_like(x), np.zeros_like(x), np.zeros_like(y))


def _camera_motion(scene: Scene, frame: int):
    ax = np.asarray(scene.camera_axis, dtype=np.float64)
    ax = ax / np.linalg.norm(ax)
    ang = np.deg2rad(scene.camera_rotation_deg) * frame * scene.frame_step
    R = quat_to_matrix(quat_from_axis_angle(ax * ang))
    t = np.asarray(scene.camera_translation, dtype=np.float64) * frame * scene.frame_step
    center = np.array([0.0, 0.0, PATCH_DISTANCE])
    return R, t + center - R @ center   # rotate about the patch centre


def make_template(scene: Scene) -> Template:
    n = scene.resolution
    L = scene.extent
    xs = np.linspace(-L / 2.0, L / 2.0, n)
    X, Y = np.meshgrid(xs, xs)
    h, gx, gy = _rest(scene)(X, Y)
    pts = np.stack([X, Y, PATCH_DISTANCE + h], axis=-1).reshape(-1, 3)
    nrm = np.stack([gx, gy, -np.ones_like(gx)], axis=-1).reshape(-1, 3)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    return Template(points=pts, normals=nrm)


def truth_points(scene: Scene, template: Template, frame: int) -> np.ndarray:
    dz, _, _ = _disp(scene, frame)(template.points[:, 0], template.points[:, 1])
    p = template.points.copy()
    p[:, 2] += dz
    R, t = _camera_motion(scene, frame)
    return p @ R.T + t


def render_depth(scene: Scene, camera: PinholeCamera, frame: int, newton_iters: int = 40):
    """Depth of the deformed, camera-moved surface by Newton iteration on each pixel ray."""
    rest, disp = _rest(scene), _disp(scene, frame)

    def surf(x, y):
        a, ax, ay = rest(x, y)
        b, bx, by = disp(x, y)
        return a + b, ax + bx, ay + by

    R, t = _camera_motion(scene, frame)
    v, u = np.mgrid[0:camera.height, 0:camera.width].astype(np.float64)
    ray = np.stack([(u - camera.cx) / camera.fx, (v - camera.cy) / camera.fy, np.ones_like(u)], -1)
    rd = ray @ R          # ray directions in the surface frame (R^T d)
    off = -(R.T @ t)
    s = np.full(u.shape, PATCH_DISTANCE)
    half = scene.extent / 2.0
    for _ in range(newton_iters):
        xr = s * rd[..., 0] + off[0]
        yr = s * rd[..., 1] + off[1]
        x = np.clip(xr, -half * 1.2, half * 1.2)
        y = np.clip(yr, -half * 1.2, half * 1.2)
        z = s * rd[..., 2] + off[2]
        g, gx, gy = surf(x, y)
        f = z - PATCH_DISTANCE - g
        df = rd[..., 2] - gx * rd[..., 0] - gy * rd[..., 1]
        step = f / df
        s = s - step
        # converged once every ray that can hit the patch has settled (rays far outside
        # the patch are clipped and never do; they are invalid anyway)
        on_patch = (np.abs(xr) <= half * 1.05) & (np.abs(yr) <= half * 1.05)
        if not np.any(on_patch) or np.max(np.abs(step[on_patch])) < 1e-11:
            break
    x = s * rd[..., 0] + off[0]
    y = s * rd[..., 1] + off[1]
    inside = (np.abs(x) <= half) & (np.abs(y) <= half) & (s > 0.0)
    depth = np.where(inside, s * ray[..., 2], 0.0)
    if scene.noise_sigma > 0.0:
        noise = np.random.default_rng((scene.seed, frame, 0)).normal(0.0, scene.noise_sigma,
                                                                     depth.shape)
        depth = np.where(depth > 0.0, depth + noise, 0.0)
    if scene.occlusion is not None:
        u0, v0, w, h = scene.occlusion
        depth[v0:v0 + h, u0:u0 + w] = 0.0
    return depth


@dataclass
class Features:
    """Template-side ORB features: descriptor bits and frame-0 3D points."""

    template_index: np.ndarray     # (T,) template point index of each feature
    descriptors: np.ndarray        # (T, 32) uint8
    points: np.ndarray             # (T, 3)


@dataclass
class FrameData:
    frame_id: int
    depth: np.ndarray
    truth: np.ndarray
    descriptors: np.ndarray        # (F, 32) uint8
    keypoints: np.ndarray          # (F, 2) int32 (u, v)
    match_src: np.ndarray          # (M, 3) 3D pairs for the MatchSet path
    match_dst: np.ndarray
    is_outlier: np.ndarray         # (T,) per template feature

    def observation(self, camera: PinholeCamera) -> Observation:
        return Observation.from_depth(self.depth, camera, frame_id=self.frame_id)

    def matches(self) -> MatchSet:
        return MatchSet.from_pairs(self.match_src, self.match_dst)


@dataclass
class Sequence:
    scene: Scene
    camera: PinholeCamera
    template: Template
    features: Features
    frames: list = field(default_factory=list)


def make_features(scene: Scene, template: Template) -> Features:
    rng = np.random.default_rng((scene.seed, 7))
    T = min(scene.n_features, len(template))
    idx = np.sort(rng.choice(len(template), size=T, replace=False))
    desc = rng.integers(0, 256, size=(T, 32), dtype=np.uint8)
    return Features(idx, desc, template.points[idx].copy())


def make_frame(scene: Scene, camera: PinholeCamera, template: Template, feats: Features,
               frame: int) -> FrameData:
    depth = render_depth(scene, camera, frame)
    truth = truth_points(scene, template, frame)
    rng = np.random.default_rng((scene.seed, frame, 11))
    T = feats.descriptors.shape[0]
    n_out = int(round(scene.outlier_fraction * T))
    outl = np.zeros(T, dtype=bool)
    if n_out:
        outl[rng.choice(T, size=n_out, replace=False)] = True
    # keypoints: inliers at the projected true position, outliers anywhere in the image
    tp = truth[feats.template_index]
    u = np.rint(camera.fx * tp[:, 0] / tp[:, 2] + camera.cx)
    v = np.rint(camera.fy * tp[:, 1] / tp[:, 2] + camera.cy)
    ru = rng.integers(0, camera.width, size=T)
    rv = rng.integers(0, camera.height, size=T)
    u = np.where(outl, ru, u).astype(np.int64)
    v = np.where(outl, rv, v).astype(np.int64)
    # descriptors: the template bits with a few random flips (every feature stays its own
    # nearest neighbour); distractors with fresh random bits
    desc = feats.descriptors.copy()
    flips = rng.integers(0, scene.max_bit_flips + 1, size=T)
    for i in range(T):
        if flips[i]:
            bits = rng.choice(256, size=flips[i], replace=False)
            desc[i, bits // 8] ^= (1 << (bits % 8)).astype(np.uint8)
    D = scene.n_distractors
    ddesc = rng.integers(0, 256, size=(D, 32), dtype=np.uint8)
    dkp = np.stack([rng.integers(0, camera.width, D), rng.integers(0, camera.height, D)], 1)
    all_desc = np.concatenate([desc, ddesc], axis=0)
    all_kp = np.concatenate([np.stack([u, v], 1), dkp], axis=0).astype(np.int32)
    perm = rng.permutation(T + D)
    all_desc, all_kp = all_desc[perm], all_kp[perm]
    # 3D pairs for the MatchSet path: inliers observe the truth, outliers are uniform in
    # the truth bounding box +-10 % (the reference's outlier model, synth.py:315-321)
    lo, hi = truth.min(axis=0), truth.max(axis=0)
    span = np.maximum(hi - lo, 5.0)
    dst = tp.copy()
    if n_out:
        dst[outl] = rng.uniform(lo - 0.1 * span, hi + 0.1 * span, size=(n_out, 3))
    src = feats.points.copy()
    if scene.occlusion is not None:
        u0, v0, w, h = scene.occlusion
        pu = camera.fx * dst[:, 0] / dst[:, 2] + camera.cx
        pv = camera.fy * dst[:, 1] / dst[:, 2] + camera.cy
        keep = ~((pu >= u0 - 0.5) & (pu < u0 + w - 0.5) & (pv >= v0 - 0.5) & (pv < v0 + h - 0.5))
        src, dst = src[keep], dst[keep]
    return FrameData(frame, depth, truth, all_desc, all_kp, src, dst, outl)


def make_sequence(scene: Scene, n_frames: int) -> Sequence:
    cam = camera_for(scene)
    tpl = make_template(scene)
    feats = make_features(scene, tpl)
    seq = Sequence(scene, cam, tpl, feats)
    for f in range(n_frames):
        seq.frames.append(make_frame(scene, cam, tpl, feats, f))
    return seq


# The BASELINE.json configurations, radius chosen for ~the stated
# control counts.
CONFIGS = {
    1: dict(scene=Scene(surface="plane", resolution=71, width=320, height=240,
                        amplitude=5.0, n_features=500, outlier_fraction=0.1,
                        n_distractors=200), radius=10.0, iters=5),
    2: dict(scene=Scene(surface="sphere-patch", resolution=141, width=640, height=480,
                        amplitude=5.0, n_features=2000, outlier_fraction=0.1), radius=5.2,
            iters=10),
    3: dict(scene=Scene(surface="height-field", resolution=141, width=640, height=480,
                        amplitude=10.0, frame_step=5, camera_rotation_deg=0.3,
                        camera_translation=(0.2, -0.1, 0.3), n_features=2000,
                        outlier_fraction=0.4), radius=5.3, iters=10),
    4: dict(scene=Scene(surface="plane", resolution=283, width=1280, height=720,
                        deformation="gaussian-poke", amplitude=8.0, n_features=2000,
                        outlier_fraction=0.1, occlusion=(320, 144, 640, 432)), radius=3.2,
            iters=10),
}


__all__ = ["Scene", "camera_for", "make_template", "truth_points", "render_depth", "Features",
           "FrameData", "Sequence", "make_features", "make_frame", "make_sequence", "CONFIGS"]
