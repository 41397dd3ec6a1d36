"""B200-native exact k-NN data-series search (Hercules hot path, arXiv 2212.13297).

Drop-in for the reference package ``seriesearch`` 0.1.0's index-build and
query entry points; all compute runs in libseriesearch_b200.so (sm_100a).
"""

from .build import BuildTrace, SeriesIndex, build_index, build_index_array, ingest_file
from .errors import DataFileError, DeviceError, IntegrityError, SeriesearchError, UsageError
from .persist import IndexSettings, QueryableIndex, load_index, write_index
from .pscan import brute_force_knn, knn_batch, pscan, pscan_query, scan_file
from .query import QueryConfig, QueryEngine, QueryStats, ResultSet, exact_knn

__version__ = "0.1.0"

__all__ = [
    "BuildTrace",
    "IndexSettings",
    "QueryEngine",
    "QueryableIndex",
    "SeriesIndex",
    "build_index",
    "build_index_array",
    "exact_knn",
    "ingest_file",
    "load_index",
    "write_index",
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
    "scan_file",
    "__version__",
]
