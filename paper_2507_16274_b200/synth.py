"""The reference trace generator's API (`memplan/synth.py`), regenerated
draw-for-draw by `tracegen` (input side; not on the device path)."""

from .tracegen import (
    DEFAULT_PALETTE,
    MIB,
    MOE_LAYER_STRIDE,
    MOE_TENSORS_PER_LAYER,
    PRESETS,
    SynthConfig,
    SynthConfigError,
    synth_arrays,
    synth_trace,
)

__all__ = ["DEFAULT_PALETTE", "MIB", "MOE_LAYER_STRIDE", "MOE_TENSORS_PER_LAYER", "PRESETS", "SynthConfig",
           "SynthConfigError", "synth_arrays", "synth_trace"]
