"""Exception types of the drop-in API (R/pkg/src/wadg/solver.py:27-28 and
the BlowUp of run()); re-exported by ``solver``."""


class BlowUp(Exception):
    """Discrete energy exceeded 1e6 x initial; the run is unstable."""


class ConfigError(ValueError):
    """Invalid solver configuration."""
