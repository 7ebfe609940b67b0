"""Type-level sizes ("nats") kept permanently in canonical polynomial form.

The reference keeps an expression tree and normalises on demand
(`SRC/nat.py:68-112`, SRC = /root/reference/pkg/src/dpia).  Here a size *is*
its normal form: a sorted tuple of (monomial, coefficient) terms, so equality,
hashing and dictionary keys are structural and O(#terms).  Monomials are sorted
tuples of variable names (with multiplicity); coefficients are positive ints.

Public helpers keep the reference's names (`nat`, `nat_equal`, `nat_eval`,
`nat_divide`, `nat_const_value`, `nat_free_vars`, `nat_str`) so callers ported
from the reference read the same.
"""
from __future__ import annotations

from typing import Dict, Iterable, Mapping, Optional, Tuple, Union

Mono = Tuple[str, ...]


class Nat:
    """An immutable polynomial over size variables with non-negative integer
    coefficients."""

    __slots__ = ("terms", "_hash")

    def __init__(self, terms: Iterable[Tuple[Mono, int]] = ()):
        acc: Dict[Mono, int] = {}
        for mono, c in terms:
            if c:
                key = tuple(sorted(mono))
                acc[key] = acc.get(key, 0) + c
        for mono, c in acc.items():
            if c < 0:
                raise ValueError("sizes must be non-negative polynomials")
        # canonical order: higher degree first, then lexicographic
        object.__setattr__(self, "terms", tuple(sorted(
            ((m, c) for m, c in acc.items() if c), key=lambda mc: (-len(mc[0]), mc[0]))))
        object.__setattr__(self, "_hash", hash(self.terms))

    def __setattr__(self, *_):
        raise AttributeError("Nat is immutable")

    # ------------------------------------------------------------ arithmetic
    def __add__(self, other: "NatLike") -> "Nat":
        return Nat(self.terms + nat(other).terms)

    __radd__ = __add__

    def __mul__(self, other: "NatLike") -> "Nat":
        o = nat(other)
        return Nat((m1 + m2, c1 * c2) for m1, c1 in self.terms for m2, c2 in o.terms)

    __rmul__ = __mul__

    def __eq__(self, other) -> bool:
        if isinstance(other, (int, str)):
            other = nat(other)
        return isinstance(other, Nat) and self.terms == other.terms

    def __hash__(self) -> int:
        return self._hash

    def __repr__(self) -> str:
        return f"Nat({nat_str(self)})"

    def __str__(self) -> str:
        return nat_str(self)

    # ---------------------------------------------------------------- queries
    @property
    def const(self) -> Optional[int]:
        if not self.terms:
            return 0
        if len(self.terms) == 1 and self.terms[0][0] == ():
            return self.terms[0][1]
        return None

    @property
    def free(self) -> frozenset:
        return frozenset(v for m, _ in self.terms for v in m)

    def evaluate(self, sigma: Mapping[str, int]) -> int:
        total = 0
        for mono, c in self.terms:
            v = c
            for name in mono:
                if name not in sigma:
                    raise KeyError(f"size variable {name!r} has no value")
                v *= int(sigma[name])
            total += v
        return total

    def substitute(self, name: str, value: "Nat") -> "Nat":
        out = Nat()
        for mono, c in self.terms:
            term = Nat([((), c)])
            for v in mono:
                term = term * (value if v == name else Nat([((v,), 1)]))
            out = out + term
        return out


NatLike = Union[Nat, int, str]
# the reference calls the abstract base NatExpr; keep the alias for callers
NatExpr = Nat


def nat(x: NatLike) -> Nat:
    if isinstance(x, Nat):
        return x
    if isinstance(x, bool):
        raise TypeError("bool is not a size")
    if isinstance(x, int):
        if x < 0:
            raise ValueError("nat constants must be non-negative")
        return Nat([((), x)])
    if isinstance(x, str):
        return Nat([((x,), 1)])
    raise TypeError(f"cannot coerce {x!r} to a size")


def nat_equal(a: NatLike, b: NatLike) -> bool:
    return nat(a) == nat(b)


def nat_normalize(e: NatLike) -> Nat:
    return nat(e)


def nat_eval(e: NatLike, sigma: Mapping[str, int]) -> int:
    return nat(e).evaluate(sigma)


def nat_const_value(e: NatLike) -> Optional[int]:
    return nat(e).const


def nat_free_vars(e: NatLike) -> frozenset:
    return nat(e).free


def nat_divide(e: NatLike, d: NatLike) -> Optional[Nat]:
    """Exact quotient e/d when d is a single monomial dividing every term of
    e (the rule `(split N E)` uses to infer the chunk count); else None."""
    e, d = nat(e), nat(d)
    if len(d.terms) != 1:
        return None
    dmono, dc = d.terms[0]
    out = []
    for mono, c in e.terms:
        if c % dc:
            return None
        rest = list(mono)
        for v in dmono:
            if v not in rest:
                return None
            rest.remove(v)
        out.append((tuple(rest), c // dc))
    return Nat(out)


def nat_str(e: NatLike) -> str:
    """Surface syntax that the reader parses back: 3, n, (* 4 n), (+ a b)."""
    e = nat(e)
    if not e.terms:
        return "0"

    def mono_str(mono: Mono, c: int) -> str:
        factors = ([str(c)] if c != 1 or not mono else []) + list(mono)
        s = factors[0]
        for f in factors[1:]:
            s = f"(* {s} {f})"
        return s

    parts = [mono_str(m, c) for m, c in e.terms]
    s = parts[0]
    for p in parts[1:]:
        s = f"(+ {s} {p})"
    return s


def nat_c(e: NatLike) -> str:
    """Infix C rendering (64-bit safe when wrapped by the caller)."""
    e = nat(e)
    if not e.terms:
        return "0"
    parts = []
    for mono, c in e.terms:
        factors = ([str(c)] if c != 1 or not mono else []) + list(mono)
        parts.append(" * ".join(factors))
    return " + ".join(parts)
