"""Measurement records — the types of `mltune.measurement`
(/root/reference/pkg/src/mltune/measurement.py:32-111) that the tuner API
passes around. Runners themselves are duck-typed (`measure(config,
repetitions) -> Sample`, optional `measured_times(indices, reps)`,
`runner_id`, `default_repetitions`; tuner.py:80-92)."""

from __future__ import annotations

from dataclasses import dataclass

STATUS_VALID = "valid"
STATUS_INVALID_STATIC = "invalid-static"
STATUS_INVALID_LAUNCH = "invalid-launch"
STATUS_INVALID_COMPILE = "invalid-compile"
INVALID_STATUSES = (STATUS_INVALID_STATIC, STATUS_INVALID_LAUNCH, STATUS_INVALID_COMPILE)
ALL_STATUSES = (STATUS_VALID,) + INVALID_STATUSES


@dataclass(frozen=True)
class Outcome:
    status: str
    time: float | None = None

    def __post_init__(self):
        if self.status not in ALL_STATUSES:
            raise ValueError(f"unknown outcome status {self.status!r}")
        if self.status == STATUS_VALID:
            if self.time is None or not self.time > 0:
                raise ValueError("valid outcome requires a strictly positive time")
        elif self.time is not None:
            raise ValueError("invalid outcome cannot carry a time")

    @classmethod
    def valid(cls, time: float) -> "Outcome":
        return cls(STATUS_VALID, float(time))

    @classmethod
    def invalid(cls, status: str) -> "Outcome":
        return cls(status, None)

    @property
    def is_valid(self) -> bool:
        return self.status == STATUS_VALID


@dataclass(frozen=True)
class Sample:
    config: tuple
    outcome: Outcome
    repetitions: int = 1
    timestamp: float | None = None

    def __post_init__(self):
        if self.outcome.is_valid and self.repetitions < 1:
            raise ValueError("valid samples require repetitions >= 1")


@dataclass(frozen=True)
class SampleSet:
    space: object
    runner_id: str
    samples: tuple

    def __post_init__(self):
        object.__setattr__(self, "samples", tuple(self.samples))
        for s in self.samples:
            self.space.validate_config(s.config)

    @property
    def space_name(self) -> str:
        return self.space.name

    def __len__(self) -> int:
        return len(self.samples)

    def valid_samples(self) -> list:
        return [s for s in self.samples if s.outcome.is_valid]
