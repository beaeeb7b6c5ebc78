"""paper_0905_2203_b200 — B200-native frequent-episode counter (arXiv 0905.2203
hot path). Counting runs only on sm_100a kernels behind the C-ABI in
include/episodic_b200.h; see DESIGN.md."""
from ._native import COUNT_PRUNED, MODE_EXACT, MODE_MINE, CSR, LIB_PATH  # noqa: F401
from .api import (  # noqa: F401
    BurstConfig, Context, DataError, Embedding, Episode, EpisodicError, Event, EventStream, GenConfig,
    IntervalConstraint, InvalidArgument, LevelResult, MiningConfig, MiningResult, Unsupported,
    count_batch, count_fsm, count_mapconcat, count_tracking, csr_to_episodes, default_context,
    find_occurrences, TrackingOptions, TrackingStats, MapConcatStats, LoadedStream, load_stream, load_stream_file, serialize_stream,
    episodes_to_csr, format_episode, generate, generate_arrays, generate_bursty_arrays, generate_candidates, mine,
    random_episodes_csr,
    validate, write_mining_csv, write_events_binary, read_events_binary,
)
