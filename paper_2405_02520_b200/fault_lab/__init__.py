"""Fault injection (reference fftshield.fault_lab)."""

from .bits import WIDTH_FOR, BitFlipInjector, FaultSpec, apply_fault, flip_bit

__all__ = ["WIDTH_FOR", "BitFlipInjector", "FaultSpec", "apply_fault", "flip_bit"]
