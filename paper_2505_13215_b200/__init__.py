"""B200-native (sm_100a) hybrid 3D-4D Gaussian Splatting render-and-train hot path."""
from .scene import Camera, HybridScene, sh_coeff_count, synthetic_scene, ring_camera, CONFIGS  # noqa: F401
