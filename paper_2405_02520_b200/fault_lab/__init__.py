"""Fault injection (reference fftshield.fault_lab)."""

from .bits import WIDTH_FOR, BitFlipInjector, FaultSpec, apply_fault, flip_bit
from .propagation import propagation_footprint

_CAMPAIGN = ("DEFAULT_DELTA_GRID", "RECORD_COLUMNS", "ROC_COLUMNS", "CampaignConfig",
             "CampaignResult", "RocPoint", "RunRecord", "records_csv", "roc_csv", "run_campaign")

__all__ = ["WIDTH_FOR", "BitFlipInjector", "FaultSpec", "apply_fault", "flip_bit",
           "propagation_footprint", *_CAMPAIGN]


def __getattr__(name):
    # campaign imports abft, which imports bits from this package: load lazily
    if name in _CAMPAIGN:
        from . import campaign
        return getattr(campaign, name)
    raise AttributeError(name)
