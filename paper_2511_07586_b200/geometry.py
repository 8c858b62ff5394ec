"""Host-side scene data: OBJ + material-map loader and builtin scene builders.

Mirrors the reference's boundary input layer so a scene loaded here is
byte-identical to what the reference's ``load_scene`` produces:

* ``load_scene(mesh_text, material_map_text)`` restates
  proj/src/geometry_io.cpp:23-191 (OBJ parsing with polygon fan
  triangulation and negative indices, material map with ambient / materials /
  regions, degenerate-triangle rejection, closed-manifold parity walk of every
  dielectric region) and Scene::finalize (proj/src/geometry.cpp:146-162).
* ``builtin_scene(name, params)`` restates proj/src/scenes.cpp:155-300 and
  emits the same OBJ / JSON text.
* New generators for the BASELINE configs (dihedral grid, coated sphere,
  procedural airframe) emit text the reference loader accepts.

The scene is plain host memory (numpy arrays in the C-ABI layouts of
include/mcsbr_gpu.h); ``paper_2511_07586_b200.solver`` uploads it to the GPU.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

from ._abi import MATERIAL_DTYPE, TRIANGLE_DTYPE


class SceneError(RuntimeError):
    """Mirrors mcsbr::SceneError (proj/include/mcsbr/geometry.hpp:19-21)."""


@dataclass
class Material:
    """mcsbr::Material (proj/include/mcsbr/em_math.hpp:99-105) + optional loss."""

    eps_r: float = 1.0
    mu_r: float = 1.0
    is_pec: bool = False
    eps_i: float = 0.0  # GPU-only extension: eps = eps_r - j*eps_i (e^{+jwt})

    def index(self) -> float:
        return 0.0 if self.is_pec else math.sqrt(self.eps_r * self.mu_r)


@dataclass
class SceneData:
    """The public data of mcsbr::Scene (geometry.hpp:55-60) after finalize()."""

    vertices: np.ndarray  # (nv, 3) float64
    triangles: np.ndarray  # (nt,) TRIANGLE_DTYPE
    materials: np.ndarray  # (nm,) MATERIAL_DTYPE, index 0 = ambient
    material_names: list = field(default_factory=list)
    eps_imag: np.ndarray | None = None  # (nm,) float64 or None (lossless)
    bounding_center: np.ndarray | None = None
    bounding_radius: float = 0.0
    diameter: float = 0.0

    @property
    def n_triangles(self) -> int:
        return len(self.triangles)

    def self_intersection_epsilon(self) -> float:
        return 1e-6 * self.diameter

    def ambient_index(self) -> float:
        m = self.materials[0]
        return 0.0 if m["is_pec"] else math.sqrt(float(m["eps_r"]) * float(m["mu_r"]))

    def finalize(self) -> "SceneData":
        """Scene::finalize (geometry.cpp:146-162): bounding sphere + validation."""
        if len(self.triangles) == 0:
            raise SceneError("scene has no triangles")
        v = self.vertices
        lo = np.array([1e300, 1e300, 1e300])
        hi = np.array([-1e300, -1e300, -1e300])
        if len(v):
            lo = np.minimum(lo, v.min(axis=0))
            hi = np.maximum(hi, v.max(axis=0))
        c = (lo + hi) * 0.5
        d = v - c
        r = 0.0
        if len(v):
            # norm = sqrt((dx*dx + dy*dy) + dz*dz), same order as em_math.hpp:44,50
            r = float(np.max(np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2])))
            r = max(0.0, r)
        self.bounding_center = c
        self.bounding_radius = r
        self.diameter = 2.0 * r
        if not self.diameter > 0.0:
            raise SceneError("scene is degenerate (zero extent)")
        return self


# ---------------------------------------------------------------------------
# OBJ + material-map loader (proj/src/geometry_io.cpp)


def _stol_prefix(tok: str) -> int:
    """std::stol on the text before the first '/' (leading integer)."""
    s = tok.strip()
    i = 0
    if i < len(s) and s[i] in "+-":
        i += 1
    j = i
    while j < len(s) and s[j].isdigit():
        j += 1
    if j == i:
        raise SceneError(f"invalid face index '{tok}'")
    return int(s[:j])


def parse_obj(text: str):
    """geometry_io.cpp:23-65 -> (vertices (nv,3), faces [(a,b,c,group,line)])."""
    verts = []
    faces = []
    group = "default"
    for line_no, line in enumerate(text.splitlines(), start=1):
        parts = line.split()
        if not parts or parts[0].startswith("#"):
            continue
        tag = parts[0]
        if tag == "v":
            try:
                verts.append((float(parts[1]), float(parts[2]), float(parts[3])))
            except (IndexError, ValueError):
                raise SceneError(f"mesh line {line_no}: malformed vertex") from None
        elif tag in ("g", "o"):
            group = parts[1] if len(parts) > 1 else "default"
        elif tag == "f":
            idx = []
            for tok in parts[1:]:
                raw = _stol_prefix(tok.split("/")[0])
                if raw == 0:
                    raise SceneError(f"mesh line {line_no}: zero face index")
                resolved = raw - 1 if raw > 0 else len(verts) + raw
                if resolved < 0 or resolved >= len(verts):
                    raise SceneError(f"mesh line {line_no}: face index out of range")
                idx.append(resolved)
            if len(idx) < 3:
                raise SceneError(f"mesh line {line_no}: face needs 3+ vertices")
            for i in range(2, len(idx)):
                faces.append((idx[0], idx[i - 1], idx[i], group, line_no))
    return np.array(verts, dtype=np.float64).reshape(-1, 3), faces


def _check_region_parity(tris: np.ndarray, material_id: int, name: str) -> None:
    """geometry_io.cpp:70-97: closed, consistently oriented boundary."""
    back = tris["back_material"] == material_id
    front = (tris["front_material"] == material_id) & ~back
    sel = back | front
    if not sel.any():
        return
    v = np.stack([tris["v0"], tris["v1"], tris["v2"]], axis=1)[sel].astype(np.int64)
    flip = front[sel]
    v[flip, 1], v[flip, 2] = v[flip, 2].copy(), v[flip, 1].copy()
    s = np.concatenate([v[:, 0], v[:, 1], v[:, 2]])
    d = np.concatenate([v[:, 1], v[:, 2], v[:, 0]])
    lo = np.minimum(s, d)
    hi = np.maximum(s, d)
    sign = np.where(s < d, 1, -1)
    key = lo * (1 << 32) + hi
    order = np.argsort(key, kind="stable")
    key_s = key[order]
    sign_s = sign[order]
    uniq, start = np.unique(key_s, return_index=True)
    sums = np.add.reduceat(sign_s, start)
    if np.any(sums != 0):
        raise SceneError(
            f"dielectric region '{name}' has a non-manifold or inconsistently oriented boundary"
        )


def triangle_normals(vertices: np.ndarray, v0, v1, v2):
    """n = cross(b - a, c - a); area2 = norm(n) in the reference's op order
    (geometry_io.cpp:171-177, em_math.hpp:44-55)."""
    a = vertices[v0]
    b = vertices[v1]
    c = vertices[v2]
    e1 = b - a
    e2 = c - a
    nx = e1[:, 1] * e2[:, 2] - e1[:, 2] * e2[:, 1]
    ny = e1[:, 2] * e2[:, 0] - e1[:, 0] * e2[:, 2]
    nz = e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]
    area2 = np.sqrt(nx * nx + ny * ny + nz * nz)
    return nx, ny, nz, area2


def load_scene(mesh_text: str, material_map_text: str) -> SceneData:
    """geometry_io.cpp:101-191 + Scene::finalize."""
    verts, faces = parse_obj(mesh_text)
    try:
        mmap = json.loads(material_map_text)
    except json.JSONDecodeError as e:
        raise SceneError(f"material map: invalid JSON: {e}") from None
    if not isinstance(mmap, dict):
        raise SceneError("material map: missing 'materials' object")
    ambient_name = mmap.get("ambient", "air")
    mats = mmap.get("materials")
    if not isinstance(mats, dict):
        raise SceneError("material map: missing 'materials' object")
    if ambient_name not in mats:
        raise SceneError(f"material map: ambient material '{ambient_name}' not defined")

    materials: list[Material] = []
    names: list[str] = []
    ids: dict[str, int] = {}

    def add(name, spec):
        spec = spec if isinstance(spec, dict) else {}
        m = Material()
        m.is_pec = bool(spec.get("pec", False))
        if not m.is_pec:
            m.eps_r = float(spec.get("eps_r", 1.0))
            m.mu_r = float(spec.get("mu_r", 1.0))
            m.eps_i = float(spec.get("eps_i", 0.0))
            if (not m.eps_r > 0.0 or not m.mu_r > 0.0 or not math.isfinite(m.eps_r)
                    or not math.isfinite(m.mu_r)):
                raise SceneError(f"material '{name}': eps_r and mu_r must be positive")
        ids[name] = len(materials)
        materials.append(m)
        names.append(name)

    add(ambient_name, mats[ambient_name])
    if materials[0].is_pec:
        raise SceneError("material map: ambient material cannot be PEC")
    # nlohmann::json objects iterate in sorted key order (std::map)
    for name in sorted(mats.keys()):
        if name == ambient_name:
            continue
        add(name, mats[name])

    regions = mmap.get("regions")
    if not isinstance(regions, dict):
        raise SceneError("material map: missing 'regions' object")
    region_ids = {}
    for group in sorted(regions.keys()):
        spec = regions[group] if isinstance(regions[group], dict) else {}
        front = spec.get("front", ambient_name)
        back = spec.get("back", ambient_name)
        for nm in (front, back):
            if nm not in ids:
                raise SceneError(f"regions.{group}: unknown material '{nm}'")
        region_ids[group] = (ids[front], ids[back])

    nt = len(faces)
    tris = np.zeros(nt, dtype=TRIANGLE_DTYPE)
    if nt:
        fa = np.array([f[0] for f in faces], dtype=np.uint32)
        fb = np.array([f[1] for f in faces], dtype=np.uint32)
        fc = np.array([f[2] for f in faces], dtype=np.uint32)
        fronts = np.empty(nt, dtype=np.uint16)
        backs = np.empty(nt, dtype=np.uint16)
        for i, f in enumerate(faces):
            r = region_ids.get(f[3])
            if r is None:
                raise SceneError(f"mesh group '{f[3]}' has no region entry (line {f[4]})")
            fronts[i], backs[i] = r
        nx, ny, nz, area2 = triangle_normals(verts, fa, fb, fc)
        bad = np.nonzero(area2 < 1e-12)[0]
        if len(bad):
            i = int(bad[0])
            raise SceneError(f"degenerate triangle {i} (mesh line {faces[i][4]})")
        tris["v0"], tris["v1"], tris["v2"] = fa, fb, fc
        tris["normal"][:, 0] = nx / area2
        tris["normal"][:, 1] = ny / area2
        tris["normal"][:, 2] = nz / area2
        tris["front_material"] = fronts
        tris["back_material"] = backs
        tris["exterior_facing"] = ((fronts == 0) | (backs == 0)).astype(np.uint8)
        for mid in range(1, len(materials)):
            if not materials[mid].is_pec:
                _check_region_parity(tris, mid, names[mid])

    mat_arr = np.zeros(len(materials), dtype=MATERIAL_DTYPE)
    for i, m in enumerate(materials):
        mat_arr[i]["eps_r"] = m.eps_r
        mat_arr[i]["mu_r"] = m.mu_r
        mat_arr[i]["is_pec"] = 1 if m.is_pec else 0
    eps_i = np.array([m.eps_i for m in materials], dtype=np.float64)
    sd = SceneData(vertices=np.ascontiguousarray(verts), triangles=tris, materials=mat_arr,
                   material_names=names, eps_imag=eps_i if np.any(eps_i != 0.0) else None)
    return sd.finalize()


def load_scene_files(mesh_path: str, material_map_path: str) -> SceneData:
    try:
        with open(mesh_path) as f:
            mesh = f.read()
    except OSError:
        raise SceneError(f"cannot open file: {mesh_path}") from None
    try:
        with open(material_map_path) as f:
            mm = f.read()
    except OSError:
        raise SceneError(f"cannot open file: {material_map_path}") from None
    return load_scene(mesh, mm)


# ---------------------------------------------------------------------------
# Mesh builder + builtin scenes (proj/src/scenes.cpp)


def _normalized(p):
    n = math.sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2])
    return (p[0] / n, p[1] / n, p[2] / n)


class MeshBuilder:
    """scenes.cpp:16-125 (vertex/tri/quad/box/plate/icosphere, OBJ writer)."""

    def __init__(self):
        self.vertices: list[tuple] = []
        self.faces: list[tuple] = []  # (a, b, c, group)

    def vertex(self, v) -> int:
        self.vertices.append((float(v[0]), float(v[1]), float(v[2])))
        return len(self.vertices) - 1

    def tri(self, a, b, c, group):
        self.faces.append((a, b, c, group))

    def quad(self, a, b, c, d, group):
        self.tri(a, b, c, group)
        self.tri(a, c, d, group)

    def box(self, lo, hi, group, skip_bottom=False):
        v000 = self.vertex((lo[0], lo[1], lo[2]))
        v100 = self.vertex((hi[0], lo[1], lo[2]))
        v010 = self.vertex((lo[0], hi[1], lo[2]))
        v110 = self.vertex((hi[0], hi[1], lo[2]))
        v001 = self.vertex((lo[0], lo[1], hi[2]))
        v101 = self.vertex((hi[0], lo[1], hi[2]))
        v011 = self.vertex((lo[0], hi[1], hi[2]))
        v111 = self.vertex((hi[0], hi[1], hi[2]))
        self.quad(v001, v101, v111, v011, group)
        if not skip_bottom:
            self.quad(v000, v010, v110, v100, group)
        self.quad(v100, v110, v111, v101, group)
        self.quad(v000, v001, v011, v010, group)
        self.quad(v010, v011, v111, v110, group)
        self.quad(v000, v100, v101, v001, group)

    def rect_plate(self, center, size_a, size_b, group):
        ha, hb = 0.5 * size_a, 0.5 * size_b
        a = self.vertex((center[0] + -ha, center[1] + -hb, center[2] + 0.0))
        b = self.vertex((center[0] + ha, center[1] + -hb, center[2] + 0.0))
        c = self.vertex((center[0] + ha, center[1] + hb, center[2] + 0.0))
        d = self.vertex((center[0] + -ha, center[1] + hb, center[2] + 0.0))
        self.quad(a, b, c, d, group)

    def icosphere(self, center, radius, subdivisions, group):
        t = (1.0 + math.sqrt(5.0)) / 2.0
        pts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t),
               (0, -1, -t), (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
        pts = [_normalized((float(p[0]), float(p[1]), float(p[2]))) for p in pts]
        tris = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
                (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
                (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
        for _ in range(subdivisions):
            cache: dict = {}

            def mid(a, b):
                key = (a, b) if a < b else (b, a)
                got = cache.get(key)
                if got is not None:
                    return got
                pa, pb = pts[a], pts[b]
                pts.append(_normalized(((pa[0] + pb[0]) * 0.5, (pa[1] + pb[1]) * 0.5,
                                        (pa[2] + pb[2]) * 0.5)))
                cache[key] = len(pts) - 1
                return cache[key]

            nxt = []
            for tr in tris:
                ab = mid(tr[0], tr[1])
                bc = mid(tr[1], tr[2])
                ca = mid(tr[2], tr[0])
                nxt += [(tr[0], ab, ca), (tr[1], bc, ab), (tr[2], ca, bc), (ab, bc, ca)]
            tris = nxt
        base = len(self.vertices)
        for p in pts:  # center + radius * p
            self.vertex((center[0] + p[0] * radius, center[1] + p[1] * radius,
                         center[2] + p[2] * radius))
        for tr in tris:
            self.tri(base + tr[0], base + tr[1], base + tr[2], group)

    def to_obj(self) -> str:
        out = []
        for v in self.vertices:
            out.append("v %s %s %s\n" % tuple(_g17(x) for x in v))
        group = ""
        for f in self.faces:
            if f[3] != group:
                group = f[3]
                out.append(f"g {group}\n")
            out.append(f"f {f[0] + 1} {f[1] + 1} {f[2] + 1}\n")
        return "".join(out)

    def to_scene(self, material_map: str) -> SceneData:
        """Same result as load_scene(self.to_obj(), material_map), without the text
        round trip (%.17g round-trips doubles exactly)."""
        return load_scene(self.to_obj(), material_map)


def _g17(x: float) -> str:
    return "%.17g" % x


def materials_json(regions: str, extra_materials: str = "") -> str:
    """scenes.cpp:137-144"""
    out = '{\n  "ambient": "air",\n  "materials": {\n'
    out += '    "air": {"eps_r": 1.0, "mu_r": 1.0},\n'
    out += '    "metal": {"pec": true}'
    if extra_materials:
        out += ",\n" + extra_materials
    out += "\n  },\n  \"regions\": {\n" + regions + "\n  }\n}\n"
    return out


def dielectric(name: str, eps_r: float, eps_i: float = 0.0) -> str:
    """scenes.cpp:146-151 (+ optional eps_i, ignored by the reference loader)."""
    if eps_i:
        return '    "%s": {"eps_r": %s, "mu_r": 1.0, "eps_i": %s}' % (name, _g17(eps_r), _g17(eps_i))
    return '    "%s": {"eps_r": %s, "mu_r": 1.0}' % (name, _g17(eps_r))


BUILTIN_NAMES = ["plate", "sphere", "pec_cube", "dihedral", "glass_cube",
                 "glass_cube_pec_bottom", "nested", "airplane_stub"]


def builtin_scene_names() -> list[str]:
    return list(BUILTIN_NAMES)


def builtin_scene(name: str, params: dict | None = None) -> tuple[str, str]:
    """scenes.cpp:160-300 -> (mesh_obj, material_map) text."""
    p = dict(params or {})

    def param(k, d):
        return float(p.get(k, d))

    def center():
        return (param("center_x_m", 0.0), param("center_y_m", 0.0), param("center_z_m", 0.0))

    m = MeshBuilder()
    if name == "plate":
        m.rect_plate(center(), param("size_a_m", 1.0), param("size_b_m", 1.0), "plate")
        mm = materials_json('    "plate": {"front": "air", "back": "metal"}')
    elif name == "sphere":
        m.icosphere(center(), param("radius_m", 1.0), int(param("subdivisions", 4)), "sphere")
        mm = materials_json('    "sphere": {"front": "air", "back": "metal"}')
    elif name == "pec_cube":
        h = 0.5 * param("size_m", 3.0)
        c = center()
        m.box((c[0] - h, c[1] - h, c[2] - h), (c[0] + h, c[1] + h, c[2] + h), "cube")
        mm = materials_json('    "cube": {"front": "air", "back": "metal"}')
    elif name == "dihedral":
        l = param("size_m", 1.0)
        a0 = m.vertex((0.0, -0.5 * l, 0.0))
        a1 = m.vertex((l, -0.5 * l, 0.0))
        a2 = m.vertex((l, 0.5 * l, 0.0))
        a3 = m.vertex((0.0, 0.5 * l, 0.0))
        m.quad(a0, a1, a2, a3, "plates")
        b1 = m.vertex((0.0, -0.5 * l, l))
        b2 = m.vertex((0.0, 0.5 * l, l))
        m.quad(a0, a3, b2, b1, "plates")
        mm = materials_json('    "plates": {"front": "air", "back": "metal"}')
    elif name in ("glass_cube", "glass_cube_pec_bottom"):
        h = 0.5 * param("size_m", 3.0)
        eps = param("eps_r", 1.5)
        c = center()
        backed = name == "glass_cube_pec_bottom"
        m.box((c[0] - h, c[1] - h, c[2] - h), (c[0] + h, c[1] + h, c[2] + h), "cube", backed)
        regions = '    "cube": {"front": "air", "back": "glass"}'
        if backed:
            p0 = m.vertex((c[0] + -h, c[1] + -h, c[2] + -h))
            p1 = m.vertex((c[0] + h, c[1] + -h, c[2] + -h))
            p2 = m.vertex((c[0] + h, c[1] + h, c[2] + -h))
            p3 = m.vertex((c[0] + -h, c[1] + h, c[2] + -h))
            m.quad(p0, p1, p2, p3, "backing")
            regions += ',\n    "backing": {"front": "glass", "back": "metal"}'
        mm = materials_json(regions, dielectric("glass", eps))
    elif name == "nested":
        ho = 0.5 * param("outer_size_m", 3.0)
        hi = 0.5 * param("inner_size_m", 2.0)
        r = param("sphere_radius_m", 0.5)
        sub = int(param("subdivisions", 3))
        m.box((-ho, -ho, -ho), (ho, ho, ho), "outer")
        m.box((-hi, -hi, -hi), (hi, hi, hi), "inner")
        m.icosphere((0.0, 0.0, 0.0), r, sub, "core")
        mm = materials_json(
            '    "outer": {"front": "air", "back": "glass_outer"},\n'
            '    "inner": {"front": "glass_outer", "back": "glass_inner"},\n'
            '    "core": {"front": "glass_inner", "back": "metal"}',
            dielectric("glass_outer", param("outer_eps_r", 1.5)) + ",\n"
            + dielectric("glass_inner", param("inner_eps_r", 2.0)))
    elif name == "airplane_stub":
        span = param("span_m", 7.0)
        length = param("length_m", 7.0)
        fin_h = param("fin_height_m", 1.5)
        hl = 0.5 * length
        body_h = 0.4
        m.box((-hl, -body_h, -body_h), (hl, body_h, body_h), "airframe")

        def wing(y_in, y_out):
            le_root, te_root, le_tip, te_tip, th = 0.9, -0.5, 0.1, -0.6, 0.05
            l0 = m.vertex((le_root, y_in, -th))
            l1 = m.vertex((te_root, y_in, -th))
            l2 = m.vertex((te_tip, y_out, -th))
            l3 = m.vertex((le_tip, y_out, -th))
            u0 = m.vertex((le_root, y_in, th))
            u1 = m.vertex((te_root, y_in, th))
            u2 = m.vertex((te_tip, y_out, th))
            u3 = m.vertex((le_tip, y_out, th))
            if y_out > y_in:
                m.quad(u0, u3, u2, u1, "airframe")
                m.quad(l0, l1, l2, l3, "airframe")
                m.quad(u0, u1, l1, l0, "airframe")
                m.quad(u3, l3, l2, u2, "airframe")
                m.quad(u0, l0, l3, u3, "airframe")
                m.quad(u1, u2, l2, l1, "airframe")
            else:
                m.quad(u0, u1, u2, u3, "airframe")
                m.quad(l0, l3, l2, l1, "airframe")
                m.quad(u0, l0, l1, u1, "airframe")
                m.quad(u3, u2, l2, l3, "airframe")
                m.quad(u0, u3, l3, l0, "airframe")
                m.quad(u1, l1, l2, u2, "airframe")

        wing(0.3, 0.5 * span)
        wing(-0.3, -0.5 * span)
        th = 0.04
        z0, z1 = 0.3, body_h + fin_h
        l0 = m.vertex((-hl, -th, z0))
        l1 = m.vertex((-hl + 1.1, -th, z0))
        l2 = m.vertex((-hl + 0.9, -th, z1))
        l3 = m.vertex((-hl + 0.35, -th, z1))
        r0 = m.vertex((-hl, th, z0))
        r1 = m.vertex((-hl + 1.1, th, z0))
        r2 = m.vertex((-hl + 0.9, th, z1))
        r3 = m.vertex((-hl + 0.35, th, z1))
        m.quad(l0, l1, l2, l3, "airframe")
        m.quad(r0, r3, r2, r1, "airframe")
        m.quad(l3, l2, r2, r3, "airframe")
        m.quad(l0, l3, r3, r0, "airframe")
        m.quad(l1, r1, r2, l2, "airframe")
        m.quad(l0, r0, r1, l1, "airframe")
        eps = param("eps_r", 0.0)
        if eps > 0.0:
            mm = materials_json('    "airframe": {"front": "air", "back": "skin"}',
                                dielectric("skin", eps))
        else:
            mm = materials_json('    "airframe": {"front": "air", "back": "metal"}')
    else:
        raise ValueError(f"unknown builtin scene: {name}")
    return m.to_obj(), mm


def make_builtin_scene(name: str, params: dict | None = None) -> SceneData:
    """scenes.cpp:302-305"""
    obj, mm = builtin_scene(name, params)
    return load_scene(obj, mm)


# ---------------------------------------------------------------------------
# Generators for the BASELINE configs


def dihedral_grid(size_m: float = 0.5, n: int = 64) -> tuple[str, str]:
    """Config 2: two size x size PEC plates at 90 deg, each an n x n quad grid
    (2*n*n triangles per plate), seam along z through the origin, opening
    toward +x+y, normals into the opening (front = air, back = metal)."""
    m = MeshBuilder()
    h = 0.5 * size_m
    # plate A in the y = 0 plane (x in [0, size], z in [-h, h]), normal +y
    ids = [[m.vertex((size_m * i / n, 0.0, -h + size_m * k / n)) for k in range(n + 1)]
           for i in range(n + 1)]
    for i in range(n):
        for k in range(n):
            m.quad(ids[i][k], ids[i][k + 1], ids[i + 1][k + 1], ids[i + 1][k], "plates")
    # plate B in the x = 0 plane (y in [0, size], z in [-h, h]), normal +x
    ids = [[m.vertex((0.0, size_m * j / n, -h + size_m * k / n)) for k in range(n + 1)]
           for j in range(n + 1)]
    for j in range(n):
        for k in range(n):
            m.quad(ids[j][k], ids[j + 1][k], ids[j + 1][k + 1], ids[j][k + 1], "plates")
    return m.to_obj(), materials_json('    "plates": {"front": "air", "back": "metal"}')


def scene_from_arrays(vertices: np.ndarray, faces: np.ndarray, face_region: np.ndarray,
                      regions: list[tuple[str, str]], materials: dict,
                      ambient: str = "air") -> SceneData:
    """Build a SceneData straight from arrays (large generated meshes), with
    the same semantics as load_scene: materials ordered ambient-first then by
    sorted name (nlohmann std::map order), normals cross(b-a, c-a)/|.|,
    degenerate-triangle rejection, exterior flags and the dielectric parity
    walk (geometry_io.cpp:101-191).

    faces: (nt, 3) vertex indices; face_region: (nt,) index into `regions`,
    a list of (front_material, back_material) names; materials: name ->
    dict(eps_r=, mu_r=, eps_i=, pec=)."""
    names = [ambient] + sorted(k for k in materials if k != ambient)
    ids = {n: i for i, n in enumerate(names)}
    mats = []
    for n in names:
        spec = materials[n]
        m = Material(is_pec=bool(spec.get("pec", False)))
        if not m.is_pec:
            m.eps_r = float(spec.get("eps_r", 1.0))
            m.mu_r = float(spec.get("mu_r", 1.0))
            m.eps_i = float(spec.get("eps_i", 0.0))
        mats.append(m)
    verts = np.ascontiguousarray(vertices, dtype=np.float64)
    f = np.ascontiguousarray(faces, dtype=np.uint32)
    nt = len(f)
    reg = np.array([(ids[a], ids[b]) for a, b in regions], dtype=np.uint16).reshape(-1, 2)
    fr = reg[np.asarray(face_region)]
    tris = np.zeros(nt, dtype=TRIANGLE_DTYPE)
    nx, ny, nz, area2 = triangle_normals(verts, f[:, 0], f[:, 1], f[:, 2])
    bad = np.nonzero(area2 < 1e-12)[0]
    if len(bad):
        raise SceneError(f"degenerate triangle {int(bad[0])}")
    tris["v0"], tris["v1"], tris["v2"] = f[:, 0], f[:, 1], f[:, 2]
    tris["normal"][:, 0] = nx / area2
    tris["normal"][:, 1] = ny / area2
    tris["normal"][:, 2] = nz / area2
    tris["front_material"] = fr[:, 0]
    tris["back_material"] = fr[:, 1]
    tris["exterior_facing"] = ((fr[:, 0] == 0) | (fr[:, 1] == 0)).astype(np.uint8)
    for mid in range(1, len(mats)):
        if not mats[mid].is_pec:
            _check_region_parity(tris, mid, names[mid])
    mat_arr = np.zeros(len(mats), dtype=MATERIAL_DTYPE)
    for i, m in enumerate(mats):
        mat_arr[i]["eps_r"], mat_arr[i]["mu_r"], mat_arr[i]["is_pec"] = m.eps_r, m.mu_r, int(m.is_pec)
    eps_i = np.array([m.eps_i for m in mats])
    sd = SceneData(vertices=verts, triangles=tris, materials=mat_arr, material_names=names,
                   eps_imag=eps_i if np.any(eps_i != 0.0) else None)
    return sd.finalize()


def scene_to_text(sd: SceneData) -> tuple[str, str]:
    """Export a SceneData as OBJ + material-map JSON in the reference's formats
    (geometry_io.cpp:23-160): one OBJ group per (front, back) material pair,
    vertices printed with %.17g so they round-trip exactly."""
    tr = sd.triangles
    pairs = np.stack([tr["front_material"], tr["back_material"]], 1).astype(np.int64)
    uniq, inv = np.unique(pairs, axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    lines = ["v %s %s %s\n" % (_g17(x), _g17(y), _g17(z)) for x, y, z in sd.vertices]
    order = np.argsort(inv, kind="stable")
    cur = -1
    f = np.stack([tr["v0"], tr["v1"], tr["v2"]], 1).astype(np.int64) + 1
    for i in order:
        if inv[i] != cur:
            cur = int(inv[i])
            lines.append(f"g r{cur}\n")
        lines.append(f"f {f[i, 0]} {f[i, 1]} {f[i, 2]}\n")
    names = sd.material_names
    mats = {}
    for i, n in enumerate(names):
        m = sd.materials[i]
        if m["is_pec"]:
            mats[n] = {"pec": True}
        else:
            mats[n] = {"eps_r": float(m["eps_r"]), "mu_r": float(m["mu_r"])}
            if sd.eps_imag is not None and sd.eps_imag[i] != 0.0:
                mats[n]["eps_i"] = float(sd.eps_imag[i])
    regions = {f"r{k}": {"front": names[a], "back": names[b]} for k, (a, b) in enumerate(uniq)}
    mm = json.dumps({"ambient": names[0], "materials": mats, "regions": regions}, indent=1)
    return "".join(lines), mm


def _extrude(loops: np.ndarray, cap: bool = True):
    """Closed surface through a sequence of closed cross-section loops.

    loops: (S, L, 3) -- S stations along the part, L points per closed loop
    (listed so that the loop turns counter-clockwise seen from the last
    station looking back).  Quads join consecutive stations, fans close both
    ends.  Vertices are shared, so the surface is a closed, consistently
    oriented manifold (outward normals)."""
    S, L, _ = loops.shape
    v = loops.reshape(-1, 3)
    idx = np.arange(S * L).reshape(S, L)
    a = idx[:-1, :]
    b = idx[:-1, np.r_[1:L, 0]]
    c = idx[1:, np.r_[1:L, 0]]
    d = idx[1:, :]
    quads = np.stack([a, b, c, d], -1).reshape(-1, 4)
    faces = [np.stack([quads[:, 0], quads[:, 2], quads[:, 1]], 1),
             np.stack([quads[:, 0], quads[:, 3], quads[:, 2]], 1)]
    extra = []
    if cap:
        c0 = loops[0].mean(axis=0)
        c1 = loops[-1].mean(axis=0)
        i0, i1 = S * L, S * L + 1
        extra = [c0, c1]
        r = np.arange(L)
        rn = np.r_[1:L, 0]
        faces.append(np.stack([np.full(L, i0), idx[0, r], idx[0, rn]], 1))
        faces.append(np.stack([np.full(L, i1), idx[-1, rn], idx[-1, r]], 1))
    verts = np.concatenate([v, np.array(extra).reshape(-1, 3)]) if extra else v
    return verts, np.concatenate(faces).astype(np.int64)


def _slab_loops(stations: np.ndarray, le_x: np.ndarray, chord: np.ndarray, pos: np.ndarray,
                thick: float, n_chord: int, axis: str) -> np.ndarray:
    """Rectangular slab cross-sections (chord x thickness) at span stations.
    axis 'y': wing (span along y, thickness along z); 'z': fin (span along z,
    thickness along y)."""
    S = len(stations)
    u = np.linspace(0.0, 1.0, n_chord + 1)
    # loop: top from trailing to leading edge, then bottom from leading to trailing
    xs_top = le_x[:, None] - (1.0 - u)[None, :] * chord[:, None]
    xs_bot = le_x[:, None] - u[None, :] * chord[:, None]
    xs = np.concatenate([xs_top, xs_bot[:, 1:-1]], axis=1)
    hs = np.concatenate([np.full(n_chord + 1, 0.5 * thick), np.full(n_chord - 1, -0.5 * thick)])
    L = xs.shape[1]
    out = np.zeros((S, L, 3))
    out[..., 0] = xs
    if axis == "y":
        out[..., 1] = pos[:, None]
        out[..., 2] = hs[None, :]
    else:
        out[..., 2] = pos[:, None]
        out[..., 1] = hs[None, :]
    return out


def airframe(target_triangles: int = 200_000, seed: int = 4, dielectric_skin: bool = False):
    """Procedural airframe (BASELINE configs 4/5): a capped
    cylindrical fuselage 12 m long, 1.5 m diameter, along x (nose at +x); two
    swept trapezoidal slab wings, 10 m span, 3 m root / 1 m tip chord; a
    vertical fin 2 m tall.  dielectric_skin: wings and fin get a 2 mm
    eps 3.5-0.05j skin over a 4 mm eps 10-1.0j skin on a PEC core (three
    nested closed surfaces per part); the fuselage stays PEC.  `seed` makes
    a deterministic ±1 mm panel perturbation of the fuselage interior rings.
    Returns (SceneData, info)."""
    rng = np.random.default_rng(seed)
    n_skin = 3 if dielectric_skin else 1

    def count(sc):
        n_th, n_x = max(16, int(round(128 * sc))), max(8, int(round(390 * sc)))
        n_c, n_s = max(6, int(round(60 * sc))), max(4, int(round(150 * sc)))
        n_fc, n_fs = max(6, int(round(40 * sc))), max(4, int(round(60 * sc)))
        return (2 * n_th * n_x + 2 * n_th + n_skin * (2 * (4 * n_c * n_s + 4 * n_c)
                                                      + 4 * n_fc * n_fs + 4 * n_fc))

    scale = np.sqrt(target_triangles / 200_000.0)
    for _ in range(3):  # refine the grid scale so the mesh lands near the target
        scale *= np.sqrt(target_triangles / count(scale))
    parts_v, parts_f, parts_r = [], [], []
    regions: list[tuple[str, str]] = []

    def add(v, f, region):
        if region not in regions:
            regions.append(region)
        off = sum(len(x) for x in parts_v)
        parts_v.append(v)
        parts_f.append(f + off)
        parts_r.append(np.full(len(f), regions.index(region)))

    # fuselage: circle loops in the yz plane, stations along x (tail -> nose)
    n_th = max(16, int(round(128 * scale)))
    n_x = max(8, int(round(390 * scale)))
    x = np.linspace(-6.0, 6.0, n_x + 1)
    th = np.linspace(0.0, 2 * np.pi, n_th, endpoint=False)
    r = 0.75 * np.ones((n_x + 1, n_th))
    r[1:-1] += rng.uniform(-1e-3, 1e-3, size=(n_x - 1, n_th))
    loops = np.zeros((n_x + 1, n_th, 3))
    loops[..., 0] = x[:, None]
    loops[..., 1] = r * np.cos(th)[None, :]
    loops[..., 2] = r * np.sin(th)[None, :]
    v, f = _extrude(loops[:, ::-1, :])  # outward normals
    add(v, f, ("air", "metal"))

    skins = [(0.0, ("skin_in", "metal"))]
    if dielectric_skin:
        skins = [(0.0, ("skin_in", "metal")), (0.004, ("skin_out", "skin_in")),
                 (0.006, ("air", "skin_out"))]
    else:
        skins = [(0.0, ("air", "metal"))]

    n_c = max(6, int(round(60 * scale)))
    n_s = max(4, int(round(150 * scale)))
    for side in (1.0, -1.0):  # wings
        s = np.linspace(0.0, 1.0, n_s + 1)
        y0, y1 = 0.5, 5.0  # root buried in the fuselage (radius 0.75), tip at half span
        pos = side * (y0 + (y1 - y0) * s)
        chord_c = 3.0 - 2.0 * s
        le_c = 1.5 - 1.6 * s  # swept leading edge
        for off, reg in skins:
            lo = _slab_loops(s, le_c + off, chord_c + 2 * off, pos, 0.10 + 2 * off, n_c, "y")
            if side > 0:
                lo = lo[:, ::-1, :]  # keep outward orientation on the +y wing
            v, f = _extrude(lo)
            add(v, f, reg)
    # vertical fin at the tail
    n_fc = max(6, int(round(40 * scale)))
    n_fs = max(4, int(round(60 * scale)))
    s = np.linspace(0.0, 1.0, n_fs + 1)
    pos = 0.5 + 2.25 * s  # from inside the fuselage to 2 m above its top (0.75)
    chord_f = 2.2 - 1.2 * s
    le_f = -3.8 - 1.0 * s
    for off, reg in skins:
        lo = _slab_loops(s, le_f + off, chord_f + 2 * off, pos, 0.08 + 2 * off, n_fc, "z")
        v, f = _extrude(lo)
        add(v, f, reg)

    verts = np.concatenate(parts_v)
    faces = np.concatenate(parts_f)
    fr = np.concatenate(parts_r)
    mats = {"air": {"eps_r": 1.0}, "metal": {"pec": True}}
    if dielectric_skin:
        mats["skin_out"] = {"eps_r": 3.5, "eps_i": 0.05}
        mats["skin_in"] = {"eps_r": 10.0, "eps_i": 1.0}
    sd = scene_from_arrays(verts, faces, fr, regions, mats)
    return sd, {"triangles": len(faces), "vertices": len(verts), "regions": regions}


def coated_sphere(core_r: float = 0.5, t_inner: float = 0.010, t_outer: float = 0.005,
                  eps_inner: complex = 4.0 - 0.1j, eps_outer: complex = 2.2 - 0.01j,
                  subdivisions: int = 5, lossless: bool = False) -> tuple[str, str]:
    """Config 3: PEC core + two concentric dielectric shells, each surface an
    icosphere.  eps = eps_r - j*eps_i; lossless=True drops Im(eps) (the
    reference's real-permittivity model, used for parity runs)."""
    m = MeshBuilder()
    r1 = core_r + t_inner
    r2 = r1 + t_outer
    m.icosphere((0.0, 0.0, 0.0), r2, subdivisions, "shell_outer")
    m.icosphere((0.0, 0.0, 0.0), r1, subdivisions, "shell_inner")
    m.icosphere((0.0, 0.0, 0.0), core_r, subdivisions, "core")
    ei = 0.0 if lossless else -complex(eps_inner).imag
    eo = 0.0 if lossless else -complex(eps_outer).imag
    mm = materials_json(
        '    "shell_outer": {"front": "air", "back": "coat_outer"},\n'
        '    "shell_inner": {"front": "coat_outer", "back": "coat_inner"},\n'
        '    "core": {"front": "coat_inner", "back": "metal"}',
        dielectric("coat_outer", complex(eps_outer).real, eo) + ",\n"
        + dielectric("coat_inner", complex(eps_inner).real, ei))
    return m.to_obj(), mm
