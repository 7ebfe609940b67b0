"""Type-directed elaboration of surface forms into explicit phrases.

Size and data-type arguments of every primitive are inferred locally from the
types of already elaborated operands, exactly as the reference elaborator does
(`SRC/parser.py:294-881`): operator sections ``(+)`` mean ``lam x y. y + x``
(`:355-365`), a bare literal adopts the type the context expects, ``reduce``
infers its accumulator type from the initial value or by trying the element
type and its components (`:523-547`), and ``(mapX F)`` may appear partially
applied under ``toGlobal/toLocal/toPrivate`` (`:366-378`).

Each surface head maps to one rule in `_RULES`; unknown heads fall through to
ordinary application.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Tuple

from .dtypes import (COMM, NUM, AccT, Array, CommT, DataType, DepFnT, ExpT,
                     FnT, Idx, Num, Pair, PhraseType, ProdT, Vector,
                     is_numeric, phrase_type_equal, subst_phrase_type, var_t)
from .reader import (ParseError, SExp, Token, error_at, head_of, number_of,
                     parse_data, parse_nat, parse_phrase_type)
from .signatures import (ARITH_OPS, MAP_FAMILY, MAPI_FAMILY, NEW_SPACE,
                         PARFOR_FAMILY, PRIMITIVES, REDUCE_FAMILY, TO_SPACE,
                         UNARY_OPS, vector_prim)
from .sizes import nat, nat_divide
from .terms import (App, Lam, Lit, PairP, Phrase, Prim, Proj, TApp, TLam, Var,
                    apply_prim, fresh_name)

Typed = Tuple[Phrase, PhraseType]


def _arr_exp(sx: SExp, t: PhraseType):
    if isinstance(t, ExpT) and isinstance(t.data, Array):
        return t.data.size, t.data.elem
    raise error_at(sx, f"expected an array expression, got {t}")


def _arr_acc(sx: SExp, t: PhraseType):
    if isinstance(t, AccT) and isinstance(t.data, Array):
        return t.data.size, t.data.elem
    raise error_at(sx, f"expected an array acceptor, got {t}")


def _data(sx: SExp, t: PhraseType) -> DataType:
    if isinstance(t, ExpT):
        return t.data
    raise error_at(sx, f"expected an expression, got {t}")


def _splat_ok(d: DataType) -> bool:
    while isinstance(d, Array):
        d = d.elem
    return is_numeric(d)


def _uncurry(t: PhraseType) -> Tuple[List[PhraseType], PhraseType]:
    args = []
    while isinstance(t, FnT):
        args.append(t.arg)
        t = t.ret
    return args, t


def _arity(sx: SExp, k: int, usage: str):
    if len(sx) != k:
        raise error_at(sx, f"expected {usage}")


class Elaborator:
    def __init__(self, env: Dict[str, PhraseType]):
        self.env = env

    def _extend(self, **more) -> "Elaborator":
        return Elaborator({**self.env, **more})

    # ------------------------------------------------------- entry points
    def infer(self, sx: SExp) -> Typed:
        if isinstance(sx, Token):
            return self._atom(sx)
        if not sx:
            raise error_at(sx, "empty form")
        h = head_of(sx)
        rule = _rule_for(h) if h is not None else None
        if rule is not None:
            return rule(self, sx)
        return self._apply(sx)

    def check(self, sx: SExp, expected: PhraseType) -> Phrase:
        if isinstance(expected, FnT):
            args, ret = _uncurry(expected)
            p, got = self.check_fn(sx, args, ret_hint=ret)
            if not phrase_type_equal(got, ret):
                raise error_at(sx, f"expected result type {ret}, got {got}")
            return p
        v = number_of(sx)
        if v is not None and isinstance(expected, ExpT):
            d = expected.data
            if isinstance(d, Idx):
                b = d.bound.const
                if isinstance(v, int) and 0 <= v and (b is None or v < b):
                    return Lit(v, d)
                raise error_at(sx, f"index literal {v} out of bounds {d}")
            if is_numeric(d) or (isinstance(d, Array) and _splat_ok(d)):
                return Lit(v, d)
        p, t = self.infer(sx)
        if not phrase_type_equal(t, expected):
            raise error_at(sx, f"expected type {expected}, got {t}")
        return p

    def check_fn(self, sx: SExp, arg_types: List[PhraseType],
                 ret_hint: Optional[PhraseType] = None) -> Typed:
        """Elaborate sx as a function of arg_types; returns (phrase, result type)."""
        h = head_of(sx)
        if h in ARITH_OPS and len(sx) == 1:
            return self._section(sx, h, arg_types)
        if h in MAP_FAMILY and len(sx) == 2 and len(arg_types) == 1:
            d = _data(sx, arg_types[0])
            if not isinstance(d, Array):
                raise error_at(sx, f"({h} F) expects an array argument, got {arg_types[0]}")
            f, ft = self.check_fn(sx[1], [ExpT(d.elem)])
            d2 = _data(sx, ft)
            return apply_prim(h, [d.size, d.elem, d2], [f]), ExpT(Array(d.size, d2))
        if h == "lam":
            return self._lam_against(sx, arg_types, ret_hint)
        p, t = self.infer(sx)
        for at in arg_types:
            if not isinstance(t, FnT) or not phrase_type_equal(t.arg, at):
                raise error_at(sx, f"expected a function from {at}, got {t}")
            t = t.ret
        return p, t

    # ---------------------------------------------------------- helpers
    def _section(self, sx, op, arg_types) -> Typed:
        if len(arg_types) != 2:
            raise error_at(sx, f"section ({op}) used at wrong arity")
        elem_t, acc_t = arg_types
        d = _data(sx, acc_t)
        if not phrase_type_equal(elem_t, acc_t):
            raise error_at(sx, f"section ({op}) needs equal operand types")
        x, y = fresh_name("x"), fresh_name("y")
        body = apply_prim(op, [d], [PairP(Var(y), Var(x))])
        return Lam(x, Lam(y, body, arg_type=acc_t), arg_type=elem_t), acc_t

    def _lam_against(self, sx, arg_types, ret_hint) -> Typed:
        binders, body_sx = sx[1:-1], sx[-1]
        if len(binders) > len(arg_types):
            raise error_at(sx, "lambda has more binders than expected arguments")
        names, inner_env = [], dict(self.env)
        for b, at in zip(binders, arg_types):
            if isinstance(b, Token):
                name = b.text
            elif isinstance(b, list) and len(b) == 2 and isinstance(b[0], Token):
                name = b[0].text
                ann = parse_phrase_type(b[1])
                if not phrase_type_equal(ann, at):
                    raise error_at(b, f"annotation {ann} does not match expected {at}")
            else:
                raise error_at(b, "malformed binder")
            inner_env[name] = at
            names.append(name)
        inner = Elaborator(inner_env)
        rest = arg_types[len(binders):]
        if rest:
            body, ret = inner.check_fn(body_sx, rest, ret_hint=ret_hint)
        elif ret_hint is not None:
            body, ret = inner.check(body_sx, ret_hint), ret_hint
        else:
            body, ret = inner.infer(body_sx)
        for name, at in zip(reversed(names), reversed(arg_types[:len(binders)])):
            body = Lam(name, body, arg_type=at)
        return body, ret

    def _atom(self, tok: Token) -> Typed:
        v = number_of(tok)
        if v is not None:
            return Lit(v), ExpT(NUM)
        if tok.text in self.env:
            return Var(tok.text, span=(tok.line, tok.col)), self.env[tok.text]
        if tok.text in PRIMITIVES:
            return Prim(tok.text, span=(tok.line, tok.col)), PRIMITIVES[tok.text]
        raise ParseError(f"unbound identifier: {tok.text}", tok.line, tok.col)

    def _apply(self, sx) -> Typed:
        p, t = self.infer(sx[0])
        for a in sx[1:]:
            if not isinstance(t, FnT):
                raise error_at(sx, f"applying a non-function of type {t}")
            p, t = App(p, self.check(a, t.arg)), t.ret
        return p, t

    def _numeric_pair(self, sx, a_sx, b_sx):
        """Two operands at a common num/vec type; a bare literal adopts the
        other operand's type."""
        a_lit, b_lit = number_of(a_sx) is not None, number_of(b_sx) is not None
        if a_lit and not b_lit:
            e2, t2 = self.infer(b_sx)
            d = _data(sx, t2)
            e1 = self.check(a_sx, ExpT(d))
        elif b_lit and not a_lit:
            e1, t1 = self.infer(a_sx)
            d = _data(sx, t1)
            e2 = self.check(b_sx, ExpT(d))
        else:
            e1, t1 = self.infer(a_sx)
            e2, t2 = self.infer(b_sx)
            d, d2 = _data(sx, t1), _data(sx, t2)
            if d != d2:
                raise error_at(sx, f"operand type mismatch: {d} vs {d2}")
        if not is_numeric(d):
            raise error_at(sx, f"arithmetic at non-numeric type {d}")
        return d, e1, e2

    def _reduce_fn(self, f_sx, d1, d2, imperative: bool) -> Phrase:
        if not imperative:
            f, ft = self.check_fn(f_sx, [ExpT(d1), ExpT(d2)], ret_hint=ExpT(d2))
            if not phrase_type_equal(ft, ExpT(d2)):
                raise error_at(f_sx, f"reduction function returns {ft}, expected (exp {d2})")
            return f
        f, ft = self.check_fn(f_sx, [ExpT(d1), ExpT(d2), AccT(d2)], ret_hint=COMM)
        if not isinstance(ft, CommT):
            raise error_at(f_sx, f"expected a command body, got {ft}")
        return f

    def _reduce_operands(self, sx, f_sx, i_sx, d1, imperative: bool):
        """Accumulator type from the init when it is not a bare literal,
        otherwise the first of d1, its pair components, num that works."""
        if number_of(i_sx) is None:
            init, it = self.infer(i_sx)
            d2 = _data(i_sx, it)
            return self._reduce_fn(f_sx, d1, d2, imperative), d2, init
        tried: List[DataType] = []
        for d2 in [d1] + ([d1.fst, d1.snd] if isinstance(d1, Pair) else []) + [NUM]:
            if d2 in tried:
                continue
            tried.append(d2)
            try:
                f = self._reduce_fn(f_sx, d1, d2, imperative)
            except ParseError:
                continue
            return f, d2, self.check(i_sx, ExpT(d2))
        raise error_at(sx, "cannot infer the accumulator type; annotate the initial value "
                           "or the reduction function")

    def _command_fn(self, sx, f_sx, arg_types, what) -> Phrase:
        f, ft = self.check_fn(f_sx, arg_types, ret_hint=COMM)
        if not isinstance(ft, CommT):
            raise error_at(sx, f"{what} must be a command, got {ft}")
        return f


# ======================================================================
# one rule per surface head


def _r_lam(el: Elaborator, sx) -> Typed:
    if len(sx) < 3:
        raise error_at(sx, "malformed lam")
    anns = []
    for b in sx[1:-1]:
        if isinstance(b, list) and len(b) == 2 and isinstance(b[0], Token):
            anns.append((b[0].text, parse_phrase_type(b[1])))
        elif isinstance(b, Token):
            raise error_at(b, f"binder {b.text!r} needs a type annotation here "
                              "(write (lam (x TYPE) ...))")
        else:
            raise error_at(b, "malformed binder")
    inner = el._extend(**dict(anns))
    body, bt = inner.infer(sx[-1])
    for name, ann in reversed(anns):
        body, bt = Lam(name, body, arg_type=ann), FnT(ann, bt)
    return body, bt


def _r_tlam(el, sx) -> Typed:
    if len(sx) != 3 or not isinstance(sx[1], list) or len(sx[1]) != 2:
        raise error_at(sx, "expected (tlam (NAME KIND) BODY)")
    name, kind = sx[1][0].text, sx[1][1].text
    if kind not in ("nat", "data"):
        raise error_at(sx, f"unknown kind: {kind}")
    body, bt = el.infer(sx[2])
    return TLam(name, kind, body), DepFnT(name, kind, bt)


def _r_tapp(el, sx) -> Typed:
    if len(sx) < 3:
        raise error_at(sx, "malformed tapp")
    p, t = el.infer(sx[1])
    for a in sx[2:]:
        if not isinstance(t, DepFnT):
            raise error_at(sx, f"type application of non-polymorphic phrase: {t}")
        arg = parse_nat(a) if t.kind == "nat" else parse_data(a)
        p, t = TApp(p, arg), subst_phrase_type(t.body, t.binder, arg)
    return p, t


def _r_proj(index: int):
    def rule(el, sx) -> Typed:
        _arity(sx, 2, f"(proj{index} E)")
        p, t = el.infer(sx[1])
        if not isinstance(t, ProdT):
            raise error_at(sx, f"projection from non-product type {t}")
        return Proj(p, index), (t.fst if index == 1 else t.snd)
    return rule


def _r_let(el, sx) -> Typed:
    _arity(sx, 3, "(let E F)")
    e, et = el.infer(sx[1])
    d1 = _data(sx, et)
    f, ft = el.check_fn(sx[2], [ExpT(d1)])
    d2 = _data(sx, ft)
    return apply_prim("let", [d1, d2], [e, f]), ExpT(d2)


def _r_as(el, sx) -> Typed:
    """(as DTYPE E): E checked at (exp DTYPE); a literal becomes a splat of
    that type (extension: e.g. the zero register tile of mm)."""
    _arity(sx, 3, "(as DTYPE E)")
    d = parse_data(sx[1])
    return el.check(sx[2], ExpT(d)), ExpT(d)


def _r_tuple(el, sx) -> Typed:
    _arity(sx, 3, "(tuple P1 P2)")
    (p1, t1), (p2, t2) = el.infer(sx[1]), el.infer(sx[2])
    return PairP(p1, p2), ProdT(t1, t2)


def _r_map(el, sx) -> Typed:
    name = sx[0].text
    _arity(sx, 3, f"({name} F E)")
    e, et = el.infer(sx[2])
    n, d1 = _arr_exp(sx, et)
    f, ft = el.check_fn(sx[1], [ExpT(d1)])
    d2 = _data(sx, ft)
    return apply_prim(name, [n, d1, d2], [f, e]), ExpT(Array(n, d2))


def _r_reduce(el, sx) -> Typed:
    name = sx[0].text
    _arity(sx, 4, f"({name} F I E)")
    e, et = el.infer(sx[3])
    n, d1 = _arr_exp(sx, et)
    f, d2, init = el._reduce_operands(sx, sx[1], sx[2], d1, imperative=False)
    return apply_prim(name, [n, d1, d2], [f, init, e]), ExpT(d2)


def _r_reduce_local(el, sx) -> Typed:
    _arity(sx, 4, "(reduceLocal F I E)")
    e, et = el.infer(sx[3])
    n, d = _arr_exp(sx, et)
    f = el._reduce_fn(sx[1], d, d, imperative=False)
    return apply_prim("reduceLocal", [n, d], [f, el.check(sx[2], ExpT(d)), e]), ExpT(d)


def _r_zip(el, sx) -> Typed:
    _arity(sx, 3, "(zip E1 E2)")
    (e1, t1), (e2, t2) = el.infer(sx[1]), el.infer(sx[2])
    (n1, d1), (n2, d2) = _arr_exp(sx, t1), _arr_exp(sx, t2)
    if n1 != n2:
        raise error_at(sx, f"zip of arrays of different sizes: {n1} vs {n2}")
    return apply_prim("zip", [n1, d1, d2], [e1, e2]), ExpT(Array(n1, Pair(d1, d2)))


def _r_split(el, sx) -> Typed:
    if len(sx) == 4:
        n, m, e_sx = parse_nat(sx[1]), parse_nat(sx[2]), sx[3]
    elif len(sx) == 3:
        n, m, e_sx = parse_nat(sx[1]), None, sx[2]
    else:
        raise error_at(sx, "expected (split N E) or (split N M E)")
    e, et = el.infer(e_sx)
    size, d = _arr_exp(sx, et)
    if m is None:
        m = nat_divide(size, n)
        if m is None:
            raise error_at(sx, f"cannot divide array size {size} into chunks of {n}; "
                               "write (split N M E)")
    elif n * m != size:
        raise error_at(sx, f"split sizes {n}*{m} do not cover {size}")
    return apply_prim("split", [n, m, d], [e]), ExpT(Array(m, Array(n, d)))


def _nested(sx, t, accept: bool):
    n, row = (_arr_acc if accept else _arr_exp)(sx, t)
    if not isinstance(row, Array):
        raise error_at(sx, f"{sx[0].text} of a non-nested array: {t}")
    return n, row


def _r_join(el, sx) -> Typed:
    _arity(sx, 2, "(join E)")
    e, et = el.infer(sx[1])
    n, row = _nested(sx, et, False)
    return apply_prim("join", [n, row.size, row.elem], [e]), ExpT(Array(n * row.size, row.elem))


def _r_transpose(el, sx) -> Typed:
    _arity(sx, 2, "(transpose E)")
    e, et = el.infer(sx[1])
    n, row = _nested(sx, et, False)
    return (apply_prim("transpose", [n, row.size, row.elem], [e]),
            ExpT(Array(row.size, Array(n, row.elem))))


def _r_pair(el, sx) -> Typed:
    _arity(sx, 3, "(pair E1 E2)")
    (e1, t1), (e2, t2) = el.infer(sx[1]), el.infer(sx[2])
    d1, d2 = _data(sx, t1), _data(sx, t2)
    return apply_prim("pair", [d1, d2], [e1, e2]), ExpT(Pair(d1, d2))


def _r_pair_elim(el, sx) -> Typed:
    which = sx[0].text
    _arity(sx, 2, f"({which} E)")
    e, et = el.infer(sx[1])
    d = _data(sx, et)
    if not isinstance(d, Pair):
        raise error_at(sx, f"{which} of a non-pair expression: {et}")
    return apply_prim(which, [d.fst, d.snd], [e]), ExpT(d.fst if which == "fst" else d.snd)


def _r_unary(el, sx) -> Typed:
    name = sx[0].text
    _arity(sx, 2, f"({name} E)")
    e, et = el.infer(sx[1])
    d = _data(sx, et)
    if not is_numeric(d):
        raise error_at(sx, f"{name} of non-numeric type {et}")
    return apply_prim(name, [d], [e]), et


def _r_arith(el, sx) -> Typed:
    op = sx[0].text
    _arity(sx, 3, f"({op} E1 E2)")
    d, e1, e2 = el._numeric_pair(sx, sx[1], sx[2])
    return apply_prim(op, [d], [PairP(e1, e2)]), ExpT(d)


def _r_idx(el, sx) -> Typed:
    _arity(sx, 3, "(idx E I)")
    e, et = el.infer(sx[1])
    if isinstance(et, ExpT) and isinstance(et.data, Vector):
        # lane of a vector (extension: vectors read as arrays of lanes)
        w = et.data.width
        return apply_prim(f"idxVec{w}", [], [e, el.check(sx[2], ExpT(Idx(nat(w))))]), ExpT(NUM)
    n, d = _arr_exp(sx, et)
    return apply_prim("idx", [n, d], [e, el.check(sx[2], ExpT(Idx(n)))]), ExpT(d)


def _r_vector(el, sx) -> Typed:
    name = sx[0].text
    vp = vector_prim(name)
    if vp is None or name not in PRIMITIVES:
        raise error_at(sx, f"illegal vector width in {name}")
    kind, w = vp
    _arity(sx, 2, f"({name} E)")
    e, et = el.infer(sx[1])

    def chunks(size, d):
        if not isinstance(d, Num):
            raise error_at(sx, f"vector reshape needs num elements, got {d}")
        m = nat_divide(size, w)
        if m is None:
            raise error_at(sx, f"array size {size} is not divisible by {w}")
        return m

    def vec_elems(d):
        if d != Vector(w):
            raise error_at(sx, f"{name} expects (vec {w}) elements, got {d}")

    if kind == "asVector":
        size, d = _arr_exp(sx, et)
        m = chunks(size, d)
        return apply_prim(name, [m], [e]), ExpT(Array(m, Vector(w)))
    if kind == "asScalar":
        m, d = _arr_exp(sx, et)
        vec_elems(d)
        return apply_prim(name, [m], [e]), ExpT(Array(m * w, NUM))
    if kind == "asVectorAcc":
        m, d = _arr_acc(sx, et)
        vec_elems(d)
        return apply_prim(name, [m], [e]), AccT(Array(m * w, NUM))
    size, d = _arr_acc(sx, et)
    m = chunks(size, d)
    return apply_prim(name, [m], [e]), AccT(Array(m, Vector(w)))


def _r_to_space(el, sx) -> Typed:
    name = sx[0].text
    _arity(sx, 3, f"({name} F E)")
    e, et = el.infer(sx[2])
    d1 = _data(sx, et)
    f, ft = el.check_fn(sx[1], [ExpT(d1)])
    d2 = _data(sx, ft)
    return App(apply_prim(name, [d1, d2], [f]), e), ExpT(d2)


def _r_seq(el, sx) -> Typed:
    if len(sx) < 3:
        raise error_at(sx, "expected (seq C1 C2 ...)")
    cs = [el.check(c, COMM) for c in sx[1:]]
    out = cs[-1]
    for c in reversed(cs[:-1]):
        out = App(Prim(";"), PairP(c, out))
    return out, COMM


def _r_assign(el, sx) -> Typed:
    _arity(sx, 3, "(:= A E)")
    a, at = el.infer(sx[1])
    if not isinstance(at, AccT):
        raise error_at(sx, f"assignment target is not an acceptor: {at}")
    return apply_prim(":=", [at.data], [PairP(a, el.check(sx[2], ExpT(at.data)))]), COMM


def _r_new(el, sx) -> Typed:
    name = sx[0].text
    _arity(sx, 3, f"({name} DTYPE F)")
    d = parse_data(sx[1])
    f = el._command_fn(sx, sx[2], [var_t(d)], f"{name} body")
    return apply_prim(name, [d], [f]), COMM


def _r_for(el, sx) -> Typed:
    _arity(sx, 3, "(for N F)")
    n = parse_nat(sx[1])
    return apply_prim("for", [n], [el._command_fn(sx, sx[2], [ExpT(Idx(n))], "for body")]), COMM


def _r_parfor(el, sx) -> Typed:
    name = sx[0].text
    _arity(sx, 3, f"({name} A F)")
    a, at = el.infer(sx[1])
    n, d = _arr_acc(sx, at)
    f = el._command_fn(sx, sx[2], [ExpT(Idx(n)), AccT(d)], f"{name} body")
    return apply_prim(name, [n, d], [a, f]), COMM


def _r_mapi(el, sx) -> Typed:
    name = sx[0].text
    _arity(sx, 4, f"({name} F E A)")
    e, et = el.infer(sx[2])
    n, d1 = _arr_exp(sx, et)
    a, at = el.infer(sx[3])
    n2, d2 = _arr_acc(sx, at)
    if n != n2:
        raise error_at(sx, f"{name} source and target sizes differ: {n} vs {n2}")
    f = el._command_fn(sx, sx[1], [ExpT(d1), AccT(d2)], f"{name} body")
    return apply_prim(name, [n, d1, d2], [f, e, a]), COMM


def _r_reducei(el, sx) -> Typed:
    _arity(sx, 5, "(reduceI F I E C)")
    e, et = el.infer(sx[3])
    n, d1 = _arr_exp(sx, et)
    f, d2, init = el._reduce_operands(sx, sx[1], sx[2], d1, imperative=True)
    c = el._command_fn(sx, sx[4], [ExpT(d2)], "reduceI consumer")
    return apply_prim("reduceI", [n, d1, d2], [f, init, e, c]), COMM


def _r_reducei_init(el, sx) -> Typed:
    _arity(sx, 5, "(reduceIInit F W E C)")
    e, et = el.infer(sx[3])
    n, d1 = _arr_exp(sx, et)
    w, wt = el.infer(sx[2])
    if not (isinstance(wt, FnT) and isinstance(wt.arg, AccT) and isinstance(wt.ret, CommT)):
        raise error_at(sx, "reduceIInit initialiser must be (lam (o (acc T)) COMMAND)")
    d2 = wt.arg.data
    f = el._reduce_fn(sx[1], d1, d2, imperative=True)
    c = el._command_fn(sx, sx[4], [ExpT(d2)], "reduceIInit consumer")
    return apply_prim("reduceIInit", [n, d1, d2], [f, w, e, c]), COMM


def _r_reducei_local(el, sx) -> Typed:
    _arity(sx, 5, "(reduceILocal F I E C)")
    e, et = el.infer(sx[3])
    n, d = _arr_exp(sx, et)
    f = el._reduce_fn(sx[1], d, d, imperative=True)
    init = el.check(sx[2], ExpT(d))
    c = el._command_fn(sx, sx[4], [ExpT(d)], "reduceILocal consumer")
    return apply_prim("reduceILocal", [n, d], [f, init, e, c]), COMM


def _r_idx_acc(el, sx) -> Typed:
    _arity(sx, 3, "(idxAcc A I)")
    a, at = el.infer(sx[1])
    n, d = _arr_acc(sx, at)
    return apply_prim("idxAcc", [n, d], [a, el.check(sx[2], ExpT(Idx(n)))]), AccT(d)


def _r_split_acc(el, sx) -> Typed:
    _arity(sx, 2, "(splitAcc A)")
    a, at = el.infer(sx[1])
    m, row = _nested(sx, at, True)
    return (apply_prim("splitAcc", [row.size, m, row.elem], [a]),
            AccT(Array(row.size * m, row.elem)))


def _r_join_acc(el, sx) -> Typed:
    _arity(sx, 3, "(joinAcc M A)")
    m = parse_nat(sx[1])
    a, at = el.infer(sx[2])
    size, d = _arr_acc(sx, at)
    n = nat_divide(size, m)
    if n is None:
        raise error_at(sx, f"cannot divide acceptor size {size} into rows of {m}")
    return apply_prim("joinAcc", [n, m, d], [a]), AccT(Array(n, Array(m, d)))


def _r_transpose_acc(el, sx) -> Typed:
    _arity(sx, 2, "(transposeAcc A)")
    a, at = el.infer(sx[1])
    m, row = _nested(sx, at, True)
    # acceptor of [m][n]d viewed as an acceptor of [n][m]d
    return (apply_prim("transposeAcc", [row.size, m, row.elem], [a]),
            AccT(Array(row.size, Array(m, row.elem))))


def _r_pair_acc(index: int):
    def rule(el, sx) -> Typed:
        name = f"pairAcc{index}"
        _arity(sx, 2, f"({name} A)")
        a, at = el.infer(sx[1])
        if not (isinstance(at, AccT) and isinstance(at.data, Pair)):
            raise error_at(sx, f"{name} of a non-pair acceptor: {at}")
        d = at.data
        return apply_prim(name, [d.fst, d.snd], [a]), AccT(d.fst if index == 1 else d.snd)
    return rule


def _r_zip_acc(index: int):
    def rule(el, sx) -> Typed:
        name = f"zipAcc{index}"
        _arity(sx, 2, f"({name} A)")
        a, at = el.infer(sx[1])
        n, d = _arr_acc(sx, at)
        if not isinstance(d, Pair):
            raise error_at(sx, f"{name} of a non-pair-array acceptor: {at}")
        return (apply_prim(name, [n, d.fst, d.snd], [a]),
                AccT(Array(n, d.fst if index == 1 else d.snd)))
    return rule


_RULES: Dict[str, Callable] = {
    "lam": _r_lam, "tlam": _r_tlam, "tapp": _r_tapp, "proj1": _r_proj(1), "proj2": _r_proj(2),
    "tuple": _r_tuple, "as": _r_as, "let": _r_let, "reduceLocal": _r_reduce_local, "zip": _r_zip, "split": _r_split,
    "join": _r_join, "transpose": _r_transpose, "pair": _r_pair, "fst": _r_pair_elim,
    "snd": _r_pair_elim, "idx": _r_idx, "seq": _r_seq, ":=": _r_assign, "for": _r_for,
    "reduceI": _r_reducei, "reduceIInit": _r_reducei_init, "reduceILocal": _r_reducei_local, "idxAcc": _r_idx_acc,
    "splitAcc": _r_split_acc, "joinAcc": _r_join_acc, "transposeAcc": _r_transpose_acc,
    "pairAcc1": _r_pair_acc(1), "pairAcc2": _r_pair_acc(2), "zipAcc1": _r_zip_acc(1),
    "zipAcc2": _r_zip_acc(2),
}
for _h in MAP_FAMILY:
    _RULES[_h] = _r_map
for _h in REDUCE_FAMILY:
    _RULES[_h] = _r_reduce
for _h in MAPI_FAMILY:
    _RULES[_h] = _r_mapi
for _h in PARFOR_FAMILY:
    _RULES[_h] = _r_parfor
for _h in TO_SPACE:
    _RULES[_h] = _r_to_space
for _h in NEW_SPACE:
    _RULES[_h] = _r_new
for _h in ARITH_OPS:
    _RULES[_h] = _r_arith
for _h in UNARY_OPS:
    _RULES[_h] = _r_unary


def _rule_for(h: str):
    rule = _RULES.get(h)
    if rule is None and vector_prim(h) is not None:
        return _r_vector
    return rule
