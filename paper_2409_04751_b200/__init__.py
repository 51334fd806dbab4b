"""B200-native Fisheye-GS rasterizer."""
from .types import (Camera, Scene, RenderOptions, RenderStats, BackwardOptions, GRAD_STRIDE, GRAD_SLICES,
                    CAMERA_FISHEYE, CAMERA_PINHOLE, CAMERA_PANORAMA)
from . import synthetic
from .api import (Rasterizer, RenderResult, ForwardContext, InvalidArgument, FgsError, render, backward,
                  split_grads, grads_as_rows)
from .build import build
