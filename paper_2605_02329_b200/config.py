"""ClusterConfig / CostProfile (mirror of slosim/engine.py:54-132).

Host-side configuration objects; :mod:`.pack` lowers them to the C-ABI structs.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field

from .domain import ConfigurationError, SLOConfig, SimTime

DEFAULT_BSZ_BUCKETS = [1, 2, 4, 8, 16, 32, 64, 128, 256]
DEFAULT_SEQ_BUCKETS = [8192 * k for k in range(1, 33)]
DEFAULT_BATCH_GROWTH = 0.03
DEFAULT_PRIOR_WEIGHT = 100
DEFAULT_DECODE_ANCHORS = [(1, 8192, 11_000), (1, 131072, 40_300)]
DEFAULT_PREFILL_ANCHOR = (131072, 8_800_000)

PREFILL_POLICY_NAMES = ("kairos-urgency", "fcfs", "sjf")
DECODE_POLICY_NAMES = ("kairos-slack", "continuous")


@dataclass
class CostProfile:
    """Where the cost models and the ground truth come from (engine.py:54-101)."""

    decode_anchors: list = field(default_factory=lambda: [tuple(a) for a in DEFAULT_DECODE_ANCHORS])
    batch_growth: float = DEFAULT_BATCH_GROWTH
    prior_weight: int = DEFAULT_PRIOR_WEIGHT
    bsz_buckets: list | None = None
    seq_buckets: list | None = None
    prefill_anchor: tuple = DEFAULT_PREFILL_ANCHOR
    prefill_gt_curve: list | None = None
    decode_noise_eps: float = 0.0
    profile_path: str | None = None

    def __post_init__(self) -> None:
        if self.decode_noise_eps < 0 or self.decode_noise_eps >= 1:
            raise ValueError("decode_noise_eps must be in [0, 1)")
        if self.prefill_anchor[0] <= 0 or self.prefill_anchor[1] <= 0:
            raise ValueError("prefill_anchor must be positive")

    def build_lut(self):
        from .costmodel import load_profile, synth_profile_from_anchors

        if self.profile_path is not None:
            lut, _ = load_profile(self.profile_path)
            return lut
        return synth_profile_from_anchors(
            self.decode_anchors,
            self.batch_growth,
            bsz_buckets=self.bsz_buckets,
            seq_buckets=self.seq_buckets,
            prior_weight=self.prior_weight,
        )

    def build_estimator(self):
        from .costmodel import PrefillThroughputEstimator, load_profile

        if self.profile_path is not None:
            _, anchor = load_profile(self.profile_path)
            return PrefillThroughputEstimator.seeded(*anchor)
        return PrefillThroughputEstimator.seeded(*self.prefill_anchor)


@dataclass
class ClusterConfig:
    """Everything one simulation needs besides the workload (engine.py:104-132)."""

    chunk_budget: int = 8192
    kv_capacity_tokens: int = 2_000_000
    transfer_base_us: SimTime = 0
    transfer_per_token_us: float = 0.0
    prefill_policy: str = "kairos-urgency"
    decode_policy: str = "kairos-slack"
    slo: SLOConfig = field(default_factory=SLOConfig)
    profile: CostProfile = field(default_factory=CostProfile)
    seed: int = 0

    def __post_init__(self) -> None:
        if self.chunk_budget < 1:
            raise ConfigurationError("chunk_budget must be >= 1")
        if self.kv_capacity_tokens < 1:
            raise ConfigurationError("kv_capacity_tokens must be >= 1")
        if self.transfer_base_us < 0 or self.transfer_per_token_us < 0:
            raise ConfigurationError("transfer delays must be >= 0")
        if self.prefill_policy not in PREFILL_POLICY_NAMES:
            raise ConfigurationError(f"unknown prefill policy {self.prefill_policy!r}")
        if self.decode_policy not in DECODE_POLICY_NAMES:
            raise ConfigurationError(f"unknown decode policy {self.decode_policy!r}")

    def to_echo_dict(self) -> dict:
        return json.loads(json.dumps(asdict(self)))
