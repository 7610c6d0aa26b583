"""B200-native VoGE render path (arXiv 2205.15401): Gaussian-ellipsoid volume
rendering forward + backward as sm_100a CUDA kernels behind a C ABI
(include/gvr_cuda.h), with this package as the host-side mirror of the
reference's ``gvr::`` render API.
"""
from .types import (  # noqa: F401
    Camera,
    GaussianScene,
    GradFlags,
    GradientBundle,
    RenderBuffers,
    SampledAttributes,
    ScalarLoss,
    SelectionConfig,
    ValidationError,
)
from .render import (  # noqa: F401
    Context,
    DeviceScene,
    Graph,
    ForwardResult,
    GvrRuntimeError,
    Tape,
    adam_step,
    backward,
    backward_into,
    backward_packed_into,
    unpack_gradients,
    backward_views_into,
    render_views_into,
    scalar_loss_views_into,
    default_context,
    render,
    render_into,
    render_with_tape,
    resynthesize,
    resynthesize_scene,
    sample_attributes,
    scalar_loss,
    scalar_loss_into,
    shade_lambert,
    normalized_weights,
    transmittance_at,
)
from .synthetic import make_bench_camera, make_bench_scene, make_orbit_camera  # noqa: F401
from .gradcheck import GradCheckEntry, GradCheckReport, gradcheck, so3_exp, so3_exp_gradient, so3_log  # noqa: F401
from .scene_io import (  # noqa: F401
    atomic_write_text, load_attrs_json, load_camera_json, load_scene_json, read_pfm, save_attrs_json,
    save_camera_json, save_scene_json, validate_camera, write_pfm)
