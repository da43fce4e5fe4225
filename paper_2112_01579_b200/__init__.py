"""B200-native fV-SRN direct volume rendering (arXiv 2112.01579).

Drop-in for the DVR hot path of the reference package ``fvsrn`` 0.1.0: the same
host API (ModelConfig / model_init / checkpoint_load, TransferFunction, Camera,
RenderSettings, ModelSource, render_image, raymarch_forward, eval_density,
decode_volume, fused_eval), with every evaluation running in hand-written
sm_100a CUDA kernels behind the C ABI of ``include/fvsrn_b200.h``.
"""

__version__ = "0.1.0"

from ._lib import CapacityError, pinned_empty, pooled_empty
from .fused import (FusedPlan, bench_compare, bench_csv, fused_eval, naive_eval_model, plan_build,
                    plan_for_model, warmup)
from .grid import (KeyframeGrids, LatentGrid, QuantizedLatentGrid, grid_dequantize, grid_init,
                   grid_quantize, grid_sample, grid_sample_backward, keyframe_bracket, keyframe_sample)
from .imaging import Camera, Image, metric_psnr, metric_ssim, png_bytes, write_png
from .model import (CheckpointError, FvsrnModel, ModelConfig, ModelForwardContext, apply_color_head,
                    apply_density_head, assemble_input, checkpoint_load, checkpoint_save,
                    color_head_backward, decode_volume, density_head_backward, eval_color,
                    eval_density, memory_footprint, model_backward, model_forward, model_init)
from .nn import (AdamState, FourierEncoder, MlpCache, MlpParams, act_eval, act_grad, adam_step,
                 fourier_encode, fourier_make, init_params, mlp_backward, mlp_eval, mlp_forward, nerf_rows)
from .render import (ModelSource, RayState, RenderSettings, VolumeSource, camera_rays, composite_invert,
                     composite_step, ray_box_intersect,
                     fibonacci_cameras, raymarch_forward, render_image, render_image_rgba8,
                     render_rays)
from .transfer import TF_PRESETS, TransferFunction, tf_eval, tf_from_json, tf_load, tf_save
from .volume import ScalarVolume, sample_volume
from .train import (ErrorGrid, ScreenTrainConfig, TemporalTrainConfig, TrainingDiverged, WorldTarget,
                    WorldTrainConfig, build_error_grid, evaluate_views, loss_csv, metrics_csv,
                    raymarch_backward, sample_world_dataset, train_screen, train_temporal, train_world)
from .device import set_devices, set_dvr_kernel, set_grid_sampler  # noqa: E402
