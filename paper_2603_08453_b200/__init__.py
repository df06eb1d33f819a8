"""B200-native LycheeCluster decode-step path (retrieval + sparse attention + lazy graft).

The compute lives in liblychee_b200.so (sm_100a CUDA behind the C ABI in
include/lychee_b200.h); this package is the host-side mirror of the
reference's tierkv retrieve/StreamState interface.
"""
from .api import (Budgets, DecodeOutcome, DeviceIndex, Engine, GraftReport, GraftSearch,  # noqa: F401
                  HostIndex, RetrievalResult, SelectionMode, StreamState, bf16_bits, bf16_round,
                  flush_take, retrieve, retrieve_ids, segment)
