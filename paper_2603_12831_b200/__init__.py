"""B200-native OmniServe serving step (arxiv 2603.12831), drop-in for the
reference package `hybridserve`'s per-layer step."""

__version__ = "0.1.0"
