"""B200-native ERX (arXiv 2408.14947) hot path: the per-line detector
pipeline behind the reference's had::ErxDetector / had::LineDetector
interface, as hand-written sm_100a CUDA behind a C ABI (include/erx_b200.h).
"""
from .detector import (ConfigError, DataError, DeviceError, Engine, ErxConfig, ErxDetector, ErxState, Error,
                       FactorizationError, FormatError, IoError, LineDetector, MetricUndefinedError, ScoredLine, SpectralLine,
                       apply_threshold, gen_lines, gen_lines_device, gen_scene_changes, gen_spec, generate_srp)
from ._lib import LIB_PATH, LibraryMissing, lib

__all__ = [
    "ConfigError", "DataError", "DeviceError", "Engine", "ErxConfig", "ErxDetector", "ErxState", "Error",
    "FactorizationError", "FormatError", "IoError", "LineDetector", "MetricUndefinedError", "ScoredLine", "SpectralLine",
    "apply_threshold", "gen_lines", "gen_lines_device", "gen_scene_changes", "gen_spec", "generate_srp", "LIB_PATH", "LibraryMissing", "lib",
]
