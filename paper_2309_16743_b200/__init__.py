"""B200-native (sm_100a) reservoir-fed online training of the heat-equation MLP
surrogate of arXiv 2309.16743 (Meyer et al.).  The product is libmel.so (C ABI,
include/mel.h, sources in csrc/); `mel` is its thin ctypes binding."""
from . import mel  # noqa: F401
from .mel import Config, Context, MelError, load_library, nccl_unique_id  # noqa: F401
