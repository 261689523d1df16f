"""Configuration dataclasses and error types of the router.

Field names, defaults and validation rules follow the reference so configs
built for ``routesim`` construct unchanged here:

* ``CostModel``     reference ``engine.py:45-101``
* ``CacheConfig``   reference ``cluster.py:31-41``
* ``PolicyConfig``  reference ``policies.py:37-67``
* ``ClusterConfig`` reference ``cluster.py:44-64``

The cost model's arithmetic (``prefill_cost_us`` / ``decode_cost_us``) is
evaluated on the device; the Python methods here exist for API parity and
for the closed-form tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

POLICY_KINDS = ("vllm", "linear", "filter", "simulate", "multiplicative", "least_bs")
# policies the device kernel scores (the north-star score plus the two
# batch-size-only ones that reuse the same fused argmin)
DEVICE_POLICY_KINDS = ("multiplicative", "vllm", "least_bs", "linear", "filter", "simulate")


class CacheFullError(Exception):
    """Pinned blocks alone exceed the configured capacity (kvcache.py:30)."""


class DuplicateRequestError(Exception):
    """Request enqueued twice on the same instance (engine.py:37)."""


class InvariantError(Exception):
    """Device state failed a consistency check (engine.py:41)."""


class NoInstancesError(Exception):
    """choose() with an empty candidate set (policies.py:33)."""


class UnsupportedConfigError(ValueError):
    """The configuration asks for a feature outside the device path."""


@dataclass(frozen=True)
class CostModel:
    prefill_base_ms: float = 5.0
    prefill_per_token_ms: float = 0.1
    decode_base_ms: float = 20.0
    decode_per_seq_ms: float = 1.0
    decode_per_ctx_token_ms: float = 0.0
    chunk_tokens: int = 2048
    max_batch_requests: int = 256

    def validate(self) -> None:
        for name in ("prefill_base_ms", "prefill_per_token_ms", "decode_base_ms",
                     "decode_per_seq_ms", "decode_per_ctx_token_ms"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be non-negative")
        if self.chunk_tokens < 1 or self.max_batch_requests < 1:
            raise ValueError("chunk_tokens and max_batch_requests must be >= 1")

    def scaled(self, factor: float) -> "CostModel":
        return replace(
            self,
            prefill_base_ms=self.prefill_base_ms * factor,
            prefill_per_token_ms=self.prefill_per_token_ms * factor,
            decode_base_ms=self.decode_base_ms * factor,
            decode_per_seq_ms=self.decode_per_seq_ms * factor,
            decode_per_ctx_token_ms=self.decode_per_ctx_token_ms * factor,
        )

    # Python's round() is round-half-even, as is the device's __double2ll_rn.
    def prefill_cost_us(self, tokens: int) -> int:
        if tokens <= 0:
            return 0
        return round((self.prefill_base_ms + self.prefill_per_token_ms * tokens) * 1000.0)

    def decode_cost_us(self, n_seqs: int, ctx_tokens: int) -> int:
        if n_seqs <= 0:
            return 0
        return round((self.decode_base_ms + self.decode_per_seq_ms * n_seqs
                      + self.decode_per_ctx_token_ms * ctx_tokens) * 1000.0)

    def step_time_us(self, prefill_tokens: int, n_decode: int, ctx_tokens: int) -> int:
        return self.prefill_cost_us(prefill_tokens) + self.decode_cost_us(n_decode, ctx_tokens)


@dataclass(frozen=True)
class CacheConfig:
    block_size: int = 16
    capacity_blocks: int | None = 40_000  # None = infinite

    def validate(self) -> None:
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")
        if self.capacity_blocks is not None and self.capacity_blocks < 1:
            raise ValueError("capacity_blocks must be >= 1 or None")


@dataclass(frozen=True)
class PolicyConfig:
    kind: str = "multiplicative"
    q_weight: float = 1.0
    kv_weight: float = 0.4
    bs_norm_cap: int | None = None
    range_threshold: int = 4
    mis_tuned: bool = False
    mis_tuned_factor: float = 4.0
    kv_indicator: str = "p_tokens"  # or "one_minus_hit"
    balance_indicator: str = "bs"  # or "total_tokens"
    tie_break_seed: int = 0

    def validate(self) -> None:
        if self.kind not in POLICY_KINDS:
            raise ValueError(f"unknown policy kind {self.kind!r}")
        if not 0.0 <= self.kv_weight <= 1.0:
            raise ValueError("kv_weight must be in [0, 1]")
        if self.range_threshold < 1:
            raise ValueError("range_threshold must be >= 1")
        if self.q_weight < 0:
            raise ValueError("q_weight must be non-negative")
        if self.kv_indicator not in ("p_tokens", "one_minus_hit"):
            raise ValueError(f"unknown kv_indicator {self.kv_indicator!r}")
        if self.balance_indicator not in ("bs", "total_tokens"):
            raise ValueError(f"unknown balance_indicator {self.balance_indicator!r}")


@dataclass(frozen=True)
class DetectorConfig:
    """Prefix-hotspot detector settings (reference detector.py:104-119)."""
    window_s: float = 60.0
    top_k_classes: int = 8
    class_key_blocks: int = 2
    consecutive_multiplier: float = 2.0
    mitigation: str = "exclude_holders"  # or "force_least_bs"
    compare_mean_non_holder: bool = False

    def validate(self) -> None:
        if self.window_s <= 0:
            raise ValueError("window_s must be positive")
        if self.top_k_classes < 1 or self.class_key_blocks < 1:
            raise ValueError("top_k_classes and class_key_blocks must be >= 1")
        if self.mitigation not in ("exclude_holders", "force_least_bs"):
            raise ValueError(f"unknown mitigation {self.mitigation!r}")


@dataclass(frozen=True)
class ClusterConfig:
    n_instances: int = 16
    cost_model: CostModel = field(default_factory=CostModel)
    cache: CacheConfig = field(default_factory=CacheConfig)
    policy: PolicyConfig = field(default_factory=PolicyConfig)
    detector: DetectorConfig | None = None
    staleness_ms: float = 0.0
    seed: int = 0
    debug_checks: bool = False
    parallel_instances: bool = False

    def validate(self) -> None:
        if self.n_instances < 1:
            raise ValueError("n_instances must be >= 1")
        if self.staleness_ms < 0:
            raise ValueError("staleness_ms must be >= 0")
        self.cost_model.validate()
        self.cache.validate()
        self.policy.validate()
        if self.detector is not None:
            self.detector.validate()

    def check_device_supported(self) -> None:
        """Reject the reference features that are outside the device path
        (SURVEY.md section 8f); every policy, staleness and the detector run on it."""
        if self.policy.kind not in DEVICE_POLICY_KINDS:
            raise UnsupportedConfigError(
                f"policy {self.policy.kind!r} is not on the device path "
                f"(supported: {', '.join(DEVICE_POLICY_KINDS)})")

