"""B200-native TASER mini-batch generation (drop-in for tgadapt's hot path).

The public names mirror ``tgadapt/__init__.py`` (reference src/__init__.py:3-23)
for the functions on the mini-batch-generation path.  All compute runs in
hand-written sm_100a kernels of libtaser_b200.so (include/taser_b200.h).
The library is mapped on first use (``_lib.load()``); if it is missing that
first call raises ImportError -- there is no CPU fallback.
"""

from ._lib import ConfigError, DataError
from .cache import (CacheState, EpochStats, cache_report, lookup, make_cache, maybe_replace, oracle_cache,
                    run_trace)
from .finder import (NeighborQuery, Neighborhood, batch_find, batch_find_arrays, find_recent, find_uniform,
                     pivot)
from .graph import TemporalGraph, build_graph, graphs_equal, temporal_neighborhood_size
from .pipeline import MiniBatchGenerator, PathConfig
from .encoders import EncoderConfig, encode_neighborhood_batch, encode_target_batch
from .sampler import PolicyOutput, SamplerConfig, decode_policy, mixer_transform, sample_without_replacement
from .scoring import SamplerGrad, score_policy, update_sampler
from .seeds import derive_seed, substream
from .selector import ImportanceScores, init_scores, select_batch, update_scores
from .surrogate import (SurrogateGrad, graphmixer_message_coefficients, graphmixer_sample_coefficients,
                        sample_loss_graphmixer, sample_loss_tgat, surrogate_grad, tgat_sample_coefficients)
from .ingest import ingest_events, load_manifest
from .matio import load_features, load_features_device, save_features

__version__ = "0.1.0"
