"""Asynchronous-iteration schedules, traces and audit (reference:
pintlab/async_engine.py).

The reference runs asynchronous Parareal as a deterministic discrete-event
simulation: one event = one slice activation whose two predecessor readings
come from version-stamped retention buffers, with staleness drawn from a
seeded schedule (async_engine.py:197-365). This module keeps those semantics
and data types by name — ``AsyncSchedule``, ``UpdateRecord``, ``EngineView``,
``AsyncTrace``, ``update_counts``, ``validate_schedule`` — while the state,
the retention buffers and every evaluation live on the GPU
(``async_parareal.simulate_parareal_async``). The free-running multi-stream
runtime with real staleness is ``async_parareal.run_async_parareal_device``.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Callable, NamedTuple

import numpy as np

POLICY_ROUND_ROBIN = "round-robin"
POLICY_RANDOM_FAIR = "random-fair"
POLICY_ADVERSARIAL = "adversarial-stale"
POLICIES = (POLICY_ROUND_ROBIN, POLICY_RANDOM_FAIR, POLICY_ADVERSARIAL)

STOP_PREDICATE = "stop-predicate"
STOP_QUIESCENCE = "quiescence"


@dataclass
class AsyncMapping:
    """Componentwise fixed-point map read from slot-indexed predecessor
    readings (async_engine.py:83-120): ``read_set[i]`` lists the (source,
    slot) pairs component i consumes, ``persistent_slots`` maps a slot to the
    base slot whose previously consumed version it replays. Same validation
    and exceptions as the reference. ``simulate_async`` runs the Parareal
    mapping built by ``async_parareal.async_parareal_mapping`` on the GPU."""

    n_updatable: int
    arity: int
    eval_fn: Callable
    read_set: dict
    persistent_slots: dict = field(default_factory=dict)
    propagators: tuple | None = None  # (coarse, fine) for the Parareal mapping

    def __post_init__(self):
        from .errors import DimensionError
        if self.n_updatable < 1:
            raise ValueError("need at least one updatable component")
        for i in range(1, self.n_updatable + 1):
            if i not in self.read_set:
                raise ValueError(f"read_set missing component {i}")
            for source, slot in self.read_set[i]:
                if not 0 <= source <= self.n_updatable:
                    raise DimensionError(f"component {i} reads unknown source {source}")
                if not 1 <= slot <= self.arity:
                    raise DimensionError(f"component {i} uses slot {slot} > arity {self.arity}")
        for slot, base in self.persistent_slots.items():
            if base in self.persistent_slots:
                raise ValueError(f"persistent slot {slot} chained onto persistent slot {base}")
        for i in range(1, self.n_updatable + 1):
            by_slot = {slot: src for src, slot in self.read_set[i]}
            for slot, base in self.persistent_slots.items():
                if slot in by_slot and by_slot.get(base) != by_slot[slot]:
                    raise ValueError(f"component {i}: persistent slot {slot} must share its source with base slot {base}")


@dataclass(frozen=True)
class AsyncSchedule:
    """Seeded description of who updates when and how stale reads may be
    (async_engine.py:38-79). delay_bound counts source versions; the fairness
    window is n_updatable * (delay_bound + 1) events."""

    seed: int
    delay_bound: int
    policy: str = POLICY_RANDOM_FAIR
    max_events: int = 20_000

    def __post_init__(self):
        if self.delay_bound < 0:
            raise ValueError(f"delay bound must be >= 0, got {self.delay_bound}")
        if self.policy not in POLICIES:
            raise ValueError(f"unknown policy {self.policy!r}, expected one of {POLICIES}")
        if self.max_events < 1:
            raise ValueError(f"max_events must be >= 1, got {self.max_events}")

    def window(self, n_updatable: int) -> int:
        return n_updatable * (self.delay_bound + 1)

    def to_dict(self) -> dict:
        return {"seed": self.seed, "delay_bound": self.delay_bound, "policy": self.policy,
                "max_events": self.max_events}

    @classmethod
    def from_dict(cls, doc: dict) -> "AsyncSchedule":
        return cls(seed=int(doc["seed"]), delay_bound=int(doc["delay_bound"]),
                   policy=doc.get("policy", POLICY_RANDOM_FAIR), max_events=int(doc.get("max_events", 20_000)))


@dataclass(frozen=True)
class UpdateRecord:
    """One event: which component fired, what it read, what came out."""

    k_global: int
    component: int
    reads: tuple  # ((source, slot, version), ...)
    digest: str   # short hash of the produced value ("" when not recorded)
    delta: float  # max-abs change against the prior value
    frozen: bool = False


class EngineView(NamedTuple):
    """Snapshot handed to stop predicates after each event."""

    k: int
    state: object            # BlockVector (device)
    last_deltas: np.ndarray  # per component; +inf until the first update
    drained: bool            # every fresh edge has consumed the newest version


@dataclass
class AsyncTrace:
    """Record of one asynchronous run (async_engine.py:143-190)."""

    events: list
    snapshots: list
    initial: object
    per_component_counts: np.ndarray
    stop_event: int
    stop_reason: str
    schedule: AsyncSchedule
    n_updatable: int
    persistent_slots: dict
    final: object = None

    @property
    def window(self) -> int:
        return self.schedule.window(self.n_updatable)

    def state_after(self, event_index: int):
        """State once ``event_index + 1`` events have run; -1 gives the start.
        The last state is always available; intermediate ones need
        record_snapshots=True."""
        if event_index < 0:
            return self.initial
        if self.snapshots:
            return self.snapshots[event_index]
        if event_index == len(self.events) - 1 and self.final is not None:
            return self.final
        raise KeyError("intermediate states were not recorded (record_snapshots=False)")

    def version_value(self, component: int, version: int):
        if version == 0:
            return self.initial[component]
        seen = 0
        for idx, ev in enumerate(self.events):
            if ev.component == component:
                seen += 1
                if seen == version:
                    return self.state_after(idx)[component]
        raise KeyError(f"component {component} never reached version {version}")

    def to_jsonl(self) -> str:
        lines = [json.dumps({"k": ev.k_global, "component": ev.component, "reads": [list(r) for r in ev.reads],
                             "digest": ev.digest, "delta": ev.delta, "frozen": ev.frozen}, sort_keys=True)
                 for ev in self.events]
        return "\n".join(lines) + ("\n" if lines else "")


class ScheduleDriver:
    """Activation order plus per-read staleness (restates async_engine.py:197-235
    so that the same seed yields the same schedule as the reference)."""

    def __init__(self, schedule: AsyncSchedule, n_updatable: int):
        self.rng = np.random.default_rng(schedule.seed)
        self.n = n_updatable
        self.bound = schedule.delay_bound
        self.policy = schedule.policy
        self.window = schedule.window(n_updatable)
        self.last_fired = {i: i - 1 - n_updatable for i in range(1, n_updatable + 1)}

    def next_component(self, k: int) -> int:
        if self.policy == POLICY_ROUND_ROBIN:
            choice = 1 + k % self.n
        elif self.policy == POLICY_ADVERSARIAL:
            choice = self.n - k % self.n
        else:
            critical = [i for i in range(1, self.n + 1) if self.last_fired[i] + self.window - k < self.n]
            if critical:
                choice = min(critical, key=lambda i: self.last_fired[i])
            else:
                choice = int(self.rng.integers(1, self.n + 1))
        self.last_fired[choice] = k
        return choice

    def sample_staleness(self) -> int:
        if self.policy == POLICY_ADVERSARIAL:
            return self.bound
        if self.bound == 0:
            return 0
        return int(self.rng.integers(0, self.bound + 1))


@dataclass
class ScheduleValidation:
    """Finite-horizon audit result (async_engine.py:378-399)."""

    fairness_violations: list
    staleness_violations: list
    provenance_violations: list

    @property
    def ok(self) -> bool:
        return not (self.fairness_violations or self.staleness_violations or self.provenance_violations)


def validate_schedule(trace: AsyncTrace, delay_bound: int | None = None,
                      window: int | None = None) -> ScheduleValidation:
    """Replay a trace and audit fairness, bounded staleness and
    remembered-slot provenance (semantics of async_engine.py:402-459)."""
    bound = trace.schedule.delay_bound if delay_bound is None else delay_bound
    win = trace.window if window is None else window
    p = trace.n_updatable
    persistent = trace.persistent_slots
    fairness, staleness, provenance = [], [], []
    versions = [0] * (p + 1)
    prev_base: dict = {}
    for ev in trace.events:
        if ev.frozen:
            continue
        fresh_now = {}
        for source, slot, version in ev.reads:
            if slot in persistent:
                expected = prev_base.get((ev.component, persistent[slot]), 0)
                if version != expected:
                    provenance.append((ev.k_global, slot, version))
            else:
                oldest = max(versions[source] - bound, 0)
                if version < oldest or version > versions[source]:
                    staleness.append((ev.k_global, source, version, oldest))
                fresh_now[slot] = version
        for slot, version in fresh_now.items():
            if slot in persistent.values():
                prev_base[(ev.component, slot)] = version
        versions[ev.component] += 1
    fired = [ev.component for ev in trace.events]
    n = len(fired)
    flagged: set = set()
    if n >= win:
        counts = np.zeros(p + 1, dtype=int)
        for idx in range(win):
            counts[fired[idx]] += 1
        start = 0
        while True:
            for comp in range(1, p + 1):
                if counts[comp] == 0 and comp not in flagged:
                    fairness.append((start, comp))
                    flagged.add(comp)
            if start + win >= n:
                break
            counts[fired[start]] -= 1
            counts[fired[start + win]] += 1
            start += 1
    return ScheduleValidation(fairness, staleness, provenance)


def update_counts(trace: AsyncTrace) -> tuple[np.ndarray, int]:
    """Per-component update totals and their maximum kappa (async_engine.py:462-471)."""
    counts = np.asarray(trace.per_component_counts, dtype=int)
    if counts[1:].size == 0:
        return counts, 0
    return counts, int(np.max(counts[1:]))
