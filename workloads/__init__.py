"""Seeded synthetic inputs shared by the CUDA path and the oracle (no method arithmetic)."""
from .models import *  # noqa: F401,F403
from .models import CONFIGS, config, hex_tiles, SEED, PARITY_SEEDS  # noqa: F401
