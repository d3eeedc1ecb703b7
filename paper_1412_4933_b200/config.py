"""Scenario files: the reference's flat `key = value` format.

parse_config_text / parse_config follow src/config.cpp:44-157: '#' starts a
comment, blank lines are skipped, every other line must be `key = value` with
a known key, numbers must parse completely (std::from_chars: no sign prefix
other than '-', no whitespace inside, integer overflow is an error), `model`
marks the model as explicit, overrides (the CLI flags the user passed) apply
after the file in order, and the result is validated.
"""
from __future__ import annotations

import re
from dataclasses import replace

from .engine import ConfigError, ExecutorKind, Model, ScenarioConfig, validate

_INT = re.compile(r"-?[0-9]+\Z")
_UINT = re.compile(r"[0-9]+\Z")
_FLOAT = re.compile(r"-?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?\Z|-?(?:inf|infinity|nan)\Z", re.I)

_INT_KEYS = ("width", "height", "agents_per_side", "steps", "repeats", "threads")
_FLOAT_KEYS = ("d0", "sel_mu", "sel_sigma", "alpha", "beta", "rho", "tau0", "q")


def _bad_value(key: str, value: str):
    raise ConfigError(f"malformed value for key '{key}': '{value}'")


def _int(key: str, value: str, lo: int, hi: int, pattern=_INT) -> int:
    if not pattern.match(value):
        _bad_value(key, value)
    v = int(value)
    if not lo <= v <= hi:  # from_chars reports result_out_of_range
        _bad_value(key, value)
    return v


def _float(key: str, value: str) -> float:
    if not _FLOAT.match(value):
        _bad_value(key, value)
    return float(value)


def apply(cfg: ScenarioConfig, key: str, value: str) -> ScenarioConfig:
    """One `key = value` assignment (src/config.cpp:44-97)."""
    if key in _INT_KEYS:
        return replace(cfg, **{key: _int(key, value, -(2**31), 2**31 - 1)})
    if key == "seed":
        return replace(cfg, seed=_int(key, value, 0, 2**64 - 1, _UINT))
    if key in _FLOAT_KEYS:
        return replace(cfg, **{key: _float(key, value)})
    if key == "model":
        if value not in ("lem", "aco"):
            _bad_value(key, value)
        return replace(cfg, model=Model.Lem if value == "lem" else Model.Aco, model_explicit=True)
    if key == "executor":
        if value not in ("seq", "par"):
            _bad_value(key, value)
        return replace(cfg, executor=ExecutorKind.Sequential if value == "seq" else ExecutorKind.Parallel)
    if key == "out_dir":
        if not value:
            _bad_value(key, value)
        return replace(cfg, out_dir=value)
    raise ConfigError(f"unknown key '{key}'")


def _trim(s: str) -> str:
    return s.strip(" \t\r\n")


def parse_config_text(text: str, overrides: list[tuple[str, str]] = ()) -> ScenarioConfig:
    """src/config.cpp:126-144."""
    cfg = ScenarioConfig()
    for lineno, line in enumerate(text.split("\n"), 1):
        if "#" in line:
            line = line[:line.index("#")]
        line = _trim(line)
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"line {lineno} is not 'key = value'")
        eq = line.index("=")
        cfg = apply(cfg, _trim(line[:eq]), _trim(line[eq + 1:]))
    for key, value in overrides:
        cfg = apply(cfg, key, value)
    validate(cfg)
    return cfg


def parse_config(path: str, overrides: list[tuple[str, str]] = ()) -> ScenarioConfig:
    """src/config.cpp:146-157: an empty path means defaults + overrides."""
    text = ""
    if path:
        try:
            with open(path, "r", encoding="utf-8", newline="") as f:
                text = f.read()
        except OSError:
            raise ConfigError(f"cannot open config file '{path}'") from None
    return parse_config_text(text, overrides)


__all__ = ["apply", "parse_config", "parse_config_text"]
