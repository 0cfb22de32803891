"""The drop-in exposes every public name of the reference package.

The reference's export list is ``ebzip/__init__.py:22-42`` (``__all__``);
it is restated here so the test does not read ``/root/reference`` at run
time.  INTEGRATION.md's import shim (``sys.modules["ebzip"] = ...``) relies on
this: every ``from ebzip import X`` of the reference must resolve.
"""

import paper_1706_03791_b200 as ebz

REFERENCE_ALL = [
    "CompressedStream",
    "CompressionOutcome",
    "CompressorConfig",
    "ContainerError",
    "DataGrid",
    "ErrorBoundSpec",
    "IntervalSuggestion",
    "MagicError",
    "MetricsReport",
    "PayloadMismatchError",
    "TruncatedError",
    "VersionError",
    "compress",
    "compute_metrics",
    "decompress",
    "deserialize",
    "grid_range",
    "serialize",
    "__version__",
]


def test_reference_exports_present():
    missing = [n for n in REFERENCE_ALL if n not in ebz.__all__ or not hasattr(ebz, n)]
    assert missing == []
    assert ebz.__version__ == "0.1.0"


def test_reference_submodules_present():
    # the reference's importable submodules on the path (codec, core, entropy,
    # metrics, analysis) have namesakes with the public functions callers use
    from paper_1706_03791_b200 import analysis, codec, core, entropy, metrics
    for mod, names in ((codec, ["compress", "decompress", "grid_digest",
                                "CompressionOutcome", "IntervalSuggestion"]),
                       (core, ["DataGrid", "serialize", "deserialize", "grid_range"]),
                       (entropy, ["CodeLengthTable", "build_code", "encode", "decode"]),
                       (metrics, ["compute_metrics", "MetricsReport", "metrics_csv_row"]),
                       (analysis, ["generate", "best_layer_scan", "interval_sweep",
                                   "rate_distortion_sweep"])):
        for n in names:
            assert hasattr(mod, n), (mod.__name__, n)
