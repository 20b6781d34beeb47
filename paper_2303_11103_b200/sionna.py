"""Sionna-RT-named facade over the B200 path.

The north_star names Sionna RT's API: ``Scene``, ``Transmitter`` /
``Receiver``, ``PlanarArray``, ``RadioMaterial``,
``scene.compute_paths(max_depth, num_samples)``, ``paths.cir()``,
``scene.coverage_map()`` and ``paths.apply_doppler()`` (PAPER.md listings).
The reference implements the same semantics as emtrace free functions; this
module maps each name onto them (Appendix A) and runs everything through
libb200rt.  ``max_depth`` keeps the reference's meaning (number of
reflections; LOS = depth 0, SURVEY Appendix A last row).
"""

from __future__ import annotations

import math

import numpy as np

from . import channel as _ch
from . import em as _em
from . import tracer as _tr
from .bvh import build
from .scene import AntennaArray as _AntennaArray
from .scene import RadioDevice as _RadioDevice
from .scene import RadioMaterial as _RadioMaterial
from .scene import Scene as _Scene
from .scene import SceneError
from .scene import SceneObject as _SceneObject
from .scene import load_scene as _load_scene


class RadioMaterial:
    """Non-magnetic material (eps_r, sigma), optionally the ITU-style power law."""

    def __init__(self, name, relative_permittivity=1.0, conductivity=0.0, trainable=False,
                 power_law=None):
        self.name = name
        self.relative_permittivity = float(relative_permittivity)
        self.conductivity = float(conductivity)
        self.trainable = bool(trainable)
        self.power_law = tuple(power_law) if power_law is not None else None

    def _to_emtrace(self):
        if self.power_law is not None:
            return _RadioMaterial(self.name, "power_law", coeffs=self.power_law)
        return _RadioMaterial(self.name, "constant", self.relative_permittivity, self.conductivity,
                              trainable=self.trainable)


class PlanarArray(_AntennaArray):
    """Sionna's PlanarArray(num_rows, num_cols, vertical_spacing, horizontal_spacing,
    pattern, polarization) — identical fields to emtrace's AntennaArray."""

    def __init__(self, num_rows=1, num_cols=1, vertical_spacing=0.5, horizontal_spacing=0.5,
                 pattern="iso", polarization="V"):
        super().__init__(int(num_rows), int(num_cols), float(vertical_spacing),
                         float(horizontal_spacing), pattern, polarization)
        self.validate()


class _Device:
    kind = ""

    def __init__(self, name, position, orientation=(0.0, 0.0, 0.0), velocity=(0.0, 0.0, 0.0)):
        self.name = name
        self.position = np.asarray(position, dtype=np.float64)
        self.orientation = tuple(float(x) for x in orientation)
        self.velocity = np.asarray(velocity, dtype=np.float64)

    def look_at(self, target):
        """Boresight (+x) towards ``target`` (a position or another device), zero roll."""
        t = target.position if isinstance(target, _Device) else np.asarray(target, dtype=np.float64)
        d = t - self.position
        dist = float(np.linalg.norm(d))
        if dist < 1e-12:
            raise SceneError(f"device {self.name!r}: look_at target coincides with position")
        self.orientation = (math.atan2(d[1], d[0]),
                            -math.asin(max(-1.0, min(1.0, d[2] / dist))), 0.0)
        return self.orientation

    def _to_emtrace(self):
        return _RadioDevice(self.kind, self.name, self.position.copy(), self.orientation,
                            self.velocity.copy())


class Transmitter(_Device):
    kind = "tx"


class Receiver(_Device):
    kind = "rx"


class SceneObject:
    """Triangle mesh with a radio material (by name)."""

    def __init__(self, name, vertices, triangles, radio_material):
        self.name = name
        self.vertices = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
        self.triangles = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
        self.radio_material = radio_material.name if isinstance(radio_material, RadioMaterial) \
            else str(radio_material)


class Paths:
    """Result of Scene.compute_paths: path table on the device + CIR helpers."""

    def __init__(self, scene, pathset, bvh):
        self._scene = scene
        self._pathset = pathset
        self._bvh = bvh
        self._gains = None

    @property
    def paths(self):
        return self._pathset.paths

    @property
    def table(self):
        return self._pathset.table

    def _ensure_gains(self):
        if self._gains is None:
            self._gains = _em.compute_gains(self._scene, self._bvh, self._pathset)
        return self._gains

    def apply_doppler(self, sampling_frequency, num_time_steps, tx_velocities=None,
                      rx_velocities=None):
        """Time evolution a_i(t) = a_i e^{j 2 pi f_D t} (em.py:462-494)."""
        self._gains = _em.apply_doppler(self._ensure_gains(), sampling_frequency, num_time_steps,
                                        tx_velocities, rx_velocities)
        return self

    def cir(self, los=True, reflection=True, diffraction=False, scattering=False,
            normalize_delays=False):
        """(a [rx, rx_ant, tx, tx_ant, path, time], tau [rx, tx, path]) (channel.py:40-72)."""
        if diffraction or scattering:
            raise NotImplementedError("only LOS and specular reflection are modelled "
                                      "(as in the reference)")
        c = _ch.build_cir(self._ensure_gains(), los=los, reflection=reflection,
                          normalize_delays=normalize_delays)
        return c.a, c.tau


class Scene:
    """Sionna-style scene container; compiles to an emtrace-compatible Scene."""

    def __init__(self, frequency=3.5e9, synthetic_array=True):
        self.frequency = float(frequency)
        self.synthetic_array = bool(synthetic_array)
        self.tx_array = PlanarArray()
        self.rx_array = PlanarArray()
        self.radio_materials = {}
        self.objects = {}
        self.transmitters = {}
        self.receivers = {}
        self._bvh = None
        self._geometry_key = None

    @property
    def wavelength(self):
        return 299792458.0 / self.frequency

    def add(self, item):
        if isinstance(item, RadioMaterial):
            self.radio_materials[item.name] = item
        elif isinstance(item, Transmitter):
            self.transmitters[item.name] = item
        elif isinstance(item, Receiver):
            self.receivers[item.name] = item
        elif isinstance(item, SceneObject):
            self.objects[item.name] = item
        else:
            raise SceneError(f"cannot add {type(item).__name__} to a scene")

    def remove(self, name):
        for d in (self.transmitters, self.receivers, self.objects, self.radio_materials):
            d.pop(name, None)

    def get(self, name):
        for d in (self.transmitters, self.receivers, self.objects, self.radio_materials):
            if name in d:
                return d[name]
        return None

    @property
    def _em(self):
        """The emtrace-compatible scene (objects, materials, arrays, devices)."""
        sc = _Scene(self.frequency,
                    [_SceneObject(o.name, o.radio_material, o.vertices, o.triangles)
                     for o in self.objects.values()],
                    {n: m._to_emtrace() for n, m in self.radio_materials.items()},
                    self.tx_array, self.rx_array,
                    [d._to_emtrace() for d in list(self.transmitters.values())
                     + list(self.receivers.values())],
                    self.synthetic_array)
        sc.validate()
        return sc

    def _accel(self, em_scene):
        key = tuple((o.name, o.radio_material, o.vertices.tobytes(), o.triangles.tobytes())
                    for o in self.objects.values()) + (tuple(self.radio_materials),)
        if self._bvh is None or key != self._geometry_key:
            self._bvh = build(em_scene)
            self._geometry_key = key
        return self._bvh

    def compute_paths(self, max_depth=3, num_samples=int(1e6), method="fibonacci", los=True,
                      reflection=True, diffraction=False, scattering=False):
        """All tx-rx paths (tracer.py:298-311): Fibonacci launch of num_samples rays per
        transmitter (or exhaustive enumeration), image method, merge, ordering."""
        if diffraction or scattering:
            raise NotImplementedError("only LOS and specular reflection are modelled "
                                      "(as in the reference)")
        em_scene = self._em
        bvh = self._accel(em_scene)
        ps = _tr.compute_paths(em_scene, bvh, int(max_depth) if reflection else 0, method=method,
                               num_rays=int(num_samples))
        if not los and ps.table is not None and ps.table.n:
            keep = (ps.table.order > 0).nonzero().flatten()
            T = ps.table
            for f in _tr.PathTable.FIELDS:
                setattr(T, f, getattr(T, f)[keep])
            ps._paths = None
        return Paths(em_scene, ps, bvh)

    def coverage_map(self, max_depth=3, num_samples=int(1e6), cm_cell_size=(1.0, 1.0),
                     cm_center=None, cm_size=None, cm_height=1.5, tx=0, method="fibonacci",
                     combining="central"):
        """Path-gain map on a horizontal grid (channel.py:236-253).

        ``cm_center``/``cm_size`` default to the scene's xy extent; ``combining``
        is the reference's tx_mode ("central" element or coherent "array")."""
        cell = cm_cell_size if np.isscalar(cm_cell_size) else cm_cell_size[0]
        if not np.isscalar(cm_cell_size) and cm_cell_size[0] != cm_cell_size[1]:
            raise ValueError("square coverage cells only (GridSpec has one cell_size)")
        em_scene = self._em
        if cm_center is None or cm_size is None:
            pts = np.concatenate([o.vertices for o in self.objects.values()] +
                                 [d.position[None] for d in self.transmitters.values()])
            lo, hi = pts.min(axis=0), pts.max(axis=0)
            cm_center = cm_center if cm_center is not None else 0.5 * (lo + hi)
            cm_size = cm_size if cm_size is not None else (hi - lo)
        nx = max(1, int(math.ceil(float(cm_size[0]) / cell)))
        ny = max(1, int(math.ceil(float(cm_size[1]) / cell)))
        origin = (float(cm_center[0]) - 0.5 * nx * cell, float(cm_center[1]) - 0.5 * ny * cell)
        grid = _ch.GridSpec(origin, float(cell), nx, ny, float(cm_height))
        tx_name = tx if isinstance(tx, str) else list(self.transmitters)[int(tx)]
        return _ch.coverage_map(em_scene, self._accel(em_scene), grid, int(max_depth),
                                method=method, num_rays=int(num_samples), tx_name=tx_name,
                                tx_mode=combining, cell_cap=2 ** 31)


def load_scene(path, frequency=None):
    """Load an emtrace .scene (JSON) file into a Sionna-style Scene."""
    em = _load_scene(path)
    sc = Scene(em.frequency_hz if frequency is None else frequency, em.synthetic_array)
    sc.tx_array = PlanarArray(**{k: getattr(em.tx_array, k) for k in
                                 ("num_rows", "num_cols", "vertical_spacing",
                                  "horizontal_spacing", "pattern", "polarization")})
    sc.rx_array = PlanarArray(**{k: getattr(em.rx_array, k) for k in
                                 ("num_rows", "num_cols", "vertical_spacing",
                                  "horizontal_spacing", "pattern", "polarization")})
    for m in em.materials.values():
        sc.add(RadioMaterial(m.name, m.eps_r, m.sigma, m.trainable,
                             m.coeffs if m.model == "power_law" else None))
    for o in em.objects:
        sc.add(SceneObject(o.name, o.vertices, o.triangles, o.material))
    for d in em.devices:
        cls = Transmitter if d.kind == "tx" else Receiver
        sc.add(cls(d.name, d.position, d.orientation, d.velocity))
    return sc
