"""B200-native exact k-NN data-series search (Hercules hot path, arXiv 2212.13297).

Drop-in for the reference package ``seriesearch`` 0.1.0's index-build and
query entry points; all compute runs in libseriesearch_b200.so (sm_100a).
"""

from .errors import DataFileError, DeviceError, IntegrityError, SeriesearchError, UsageError
from .pscan import brute_force_knn, knn_batch, pscan, pscan_query
from .query import QueryConfig, QueryStats, ResultSet

__version__ = "0.1.0"

__all__ = [
    "DataFileError",
    "DeviceError",
    "IntegrityError",
    "QueryConfig",
    "QueryStats",
    "ResultSet",
    "SeriesearchError",
    "UsageError",
    "brute_force_knn",
    "knn_batch",
    "pscan",
    "pscan_query",
    "__version__",
]
