"""`EmuConfig` — the knobs of the drop-in API (reference emulate.py:30-78).

Same fields, defaults, validation and `resolved_moduli` table as the reference.
`n_block` is honoured as a working-set bound (B is processed in column blocks of
at least 256); results are bitwise independent of it, as in the reference
(tests/test_emulate.py:90-96 there).  `strategy` is accepted for all three
reference values — they are bitwise identical by contract
(kernel.py:81-88) and the GPU always runs the Karatsuba form.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError

PRECISIONS = ("single", "double")
DOMAINS = ("real", "complex")
MODES = ("fast", "accurate")
STRATEGIES = ("karatsuba", "expand-rows", "expand-cols")
DEFAULT_N_BLOCK = 8192
MAX_K_REAL = 2 ** 17
MAX_K_COMPLEX = 2 ** 16

_DEFAULT_MODULI = {
    ("complex", "single", "fast"): 8,
    ("complex", "single", "accurate"): 7,
    ("complex", "double", "fast"): 14,
    ("complex", "double", "accurate"): 15,
    ("real", "single", "fast"): 8,
    ("real", "single", "accurate"): 7,
    ("real", "double", "fast"): 15,
    ("real", "double", "accurate"): 15,
}


@dataclass
class EmuConfig:
    """Emulation parameters; ``num_moduli=None`` picks the default for the
    precision/domain/mode combination."""

    precision: str = "double"
    domain: str = "real"
    mode: str = "fast"
    num_moduli: int | None = None
    n_block: int = DEFAULT_N_BLOCK
    strategy: str = "karatsuba"

    def __post_init__(self):
        if self.precision not in PRECISIONS:
            raise ConfigError(f"precision must be one of {PRECISIONS}")
        if self.domain not in DOMAINS:
            raise ConfigError(f"domain must be one of {DOMAINS}")
        if self.mode not in MODES:
            raise ConfigError(f"mode must be one of {MODES}")
        if self.strategy not in STRATEGIES:
            raise ConfigError(f"strategy must be one of {STRATEGIES}")
        if self.n_block < 1:
            raise ConfigError("n_block must be >= 1")
        if self.num_moduli is not None and not 1 <= self.num_moduli <= 20:
            raise ConfigError("num_moduli must be in 1..20")

    @property
    def resolved_moduli(self) -> int:
        if self.num_moduli is not None:
            return self.num_moduli
        return _DEFAULT_MODULI[(self.domain, self.precision, self.mode)]
