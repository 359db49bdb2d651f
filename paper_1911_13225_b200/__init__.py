"""B200-native DIST differentiable sphere tracing (arXiv 1911.13225).

Drop-in for the hot path of the reference package `sdftrace`: the same public
names for tracing, maps, heads, losses and the latent-code optimiser, backed
by libdist_b200.so (hand-written sm_100a kernels behind a C ABI,
include/dist.h).  There is no CPU fallback.
"""

from .autodiff import TapedEval, backward, eval_field_taped
from .camera import Camera, Intrinsics, Pose, RayBundle, generate_rays, log_rotation, look_at, \
    pose_gradient, project, rotation_derivatives, rotation_matrix, unproject
from .fields import AttributeField, NeuralField, eval_field
from .formats import load_camera, load_field, read_pfm, read_pgm, save_camera, save_field, \
    write_pfm, write_pgm
from .losses import LossWeights, Observation, bilinear_sample, depth_loss, latent_reg, \
    normal_loss, photometric_loss, silhouette_loss, to_gray, visibility_mask
from .optimize import AdamState, LatentOptimizer, OptimizationError, OptimizeReport, adam_step, \
    complete_shape, completion_objective, pose_objective, reconstruct_multiview, recover_pose
from .shading import HeadBundle, RenderMaps, attribute_map, depth_map, diff_heads, hard_mask, \
    normal_map, ray_distance, render, soft_silhouette, surface_points
from .shard import TileShard
from .tracer import CONVERGED, ESCAPED, EXHAUSTED, MARCHING, DeviceTrace, RayState, TraceConfig, \
    TraceResult, trace, trace_external, trace_views

__version__ = "0.1.0"
