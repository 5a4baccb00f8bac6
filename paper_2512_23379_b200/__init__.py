"""B200-native (sm_100a) streaming hot path of SoulX-FlashTalk (arXiv 2512.23379).

Drop-in for the reference lab `ftlk`'s denoise + decode path: the same model
config (`NetConfig`), sampler (`SamplerPlan`, `few_step_sample`), denoiser
entry points (`Denoiser.forward`, `as_denoise_fn`) and streaming engine
(`StreamConfig`, `start_stream`, `StreamSession`), executed by hand-written
tcgen05/TMA kernels in `_lib/libftb2.so` through a C ABI (include/ftb2.h).
"""

__version__ = "0.1.0"

from .config import NetConfig, NoiseSchedule, SamplerPlan, StreamConfig  # noqa: F401
from .errors import ConfigError, NumericError  # noqa: F401
