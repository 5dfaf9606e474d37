"""Oracle error classes (test infrastructure only).

The oracle raises the product's exception classes so tests can assert the same
types on both sides; the product hierarchy restates
`/root/reference/pkg/src/inferix/errors.py:4-33`.
"""

from paper_2511_20714_b200.errors import (  # noqa: F401
    CapacityError,
    ConfigError,
    DimensionError,
    InferixError,
    MaskError,
    OutOfRangeError,
)
