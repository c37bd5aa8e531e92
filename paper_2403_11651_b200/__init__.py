"""B200-native Cool-chic rate-distortion forward (arXiv 2403.11651).

The product is the C-ABI library libccrd.so (include/ccrd.h) built from
csrc/*.cu for sm_100a; ``ccrd`` is its thin ctypes binding and ``dist`` the
one-process-per-GPU sharding.  There is no CPU fallback.
"""
from . import ccrd  # noqa: F401
from .ccrd import (  # noqa: F401
    CcError, CcImageIO, CcModelDesc, CcRdResult, CcStrip, DeviceBatch, cc_arm_rate, cc_mac_per_pixel,
    cc_rd_forward, cc_rd_forward_host, cc_rd_forward_strip, cc_strip_latent_count, cc_strip_window,
    cc_synthesize, cc_upsample, cc_validate, cc_workspace_bytes, cc_workspace_bytes_host,
    cc_workspace_bytes_strip, desc_from_config, load, cc_train_param_count, cc_train_workspace_bytes,
    cc_train_step, CcAdam, DeviceTrainer, cc_decode, CcAnalysisDesc, analysis_desc, cc_analysis_param_count,
    cc_analysis_workspace_bytes, cc_analysis_forward, cc_arm_decode, cc_arm_decode_workspace_bytes,
    cc_set_arm_path, cc_get_arm_path, cc_arm_path_for, arm_path, CC_ARM_AUTO, CC_ARM_FFMA2, CC_ARM_TC,
    cc_set_synth_path, cc_get_synth_path, synth_path, CC_SYN_AUTO, CC_SYN_FFMA2, CC_SYN_MMA, CC_SYN_TMA,
)

__version__ = "0.1.0"
