"""Kernel language front-end (parse + type check) and the binding of
validated kernels to sm_100a entry points."""

from .check import KernelIR, validate
from .lang import parse_source, tokenize

__all__ = ["KernelIR", "parse_and_validate", "parse_source", "tokenize", "validate"]


def parse_and_validate(source: str) -> dict:
    """Source text -> {kernel name: KernelIR}.  Raises CompileError."""
    return {k.name: validate(k) for k in parse_source(source)}
