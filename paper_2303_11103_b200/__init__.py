"""B200-native (sm_100a) implementation of the emtrace / Sionna RT propagation hot path.

Public names mirror /root/reference/pkg/src/emtrace/__init__.py for the hot
path (BVH, paths, field transfer, CIR, coverage); the work runs in the CUDA
library ``_native/libb200rt.so`` through the C ABI in ``include/b200rt.h``.
"""

from .bvh import Bvh, Hit, build
from .channel import (ChannelError, Cir, CoverageMap, FreqResponse, GridSpec, build_cir,
                      coverage_map, frequency_response, load_cir, point_path_gain,
                      probe_receiver, save_cir, subcarrier_frequencies)
from .em import (ChannelGains, DiffComplex, EmError, EvalContext, PathGain, PathGeometry,
                 apply_doppler, compute_gains, fresnel, fresnel_batch, geometry_for_positions,
                 geometry_from_path,
                 path_geometry, path_materials, transfer)
from .scene import (AntennaArray, RadioDevice, RadioMaterial, Scene, SceneError, SceneObject,
                    load_scene, look_at, material_eta, write_scene)
from .tracer import (PathSet, PropagationPath, TracerError, compute_paths,
                     compute_paths_between, dump_paths, enumerate_candidates, image_solve,
                     launch_candidates, los_path)

__version__ = "0.1.0"
