"""Oracle (test infrastructure only): the reference's record line layout, i.e. nlohmann/json
3.11 `dump()` of the object built in proj/src/records.cpp:65-95 - keys sorted (std::map),
compact separators, doubles as the shortest round-trip digits laid out by nlohmann's
format_buffer (fixed when the decimal point position n is in (-4, 15], with ".0" on integral
values; otherwise d[.ddd]e+XX with at least two exponent digits), NaN/inf -> null, strings
escaped with ensure_ascii = false. Restated from nlohmann's serializer (third-party, not under
/root/reference; version 3.11.x per the SURVEY)."""
import math
from decimal import Decimal


def fmt_double(v: float) -> str:
    if not math.isfinite(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    neg = v < 0
    t = Decimal(repr(abs(v))).as_tuple()
    digits = "".join(map(str, t.digits)).rstrip("0") or "0"
    # value = 0.d1..dk x 10^n
    n = len(t.digits) + t.exponent
    k = len(digits)
    if k <= n <= 15:
        out = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        out = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        out = "0." + "0" * (-n) + digits
    else:
        out = digits[0] + ("." + digits[1:] if k > 1 else "")
        e = n - 1
        out += "e" + ("-" if e < 0 else "+") + ("0" if abs(e) < 10 else "") + str(abs(e))
    return ("-" if neg else "") + out


def _quote(s: str) -> str:
    out = ['"']
    for ch in s:
        c = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif ch == "\b":
            out.append("\\b")
        elif ch == "\f":
            out.append("\\f")
        elif ch == "\n":
            out.append("\\n")
        elif ch == "\r":
            out.append("\\r")
        elif ch == "\t":
            out.append("\\t")
        elif c < 0x20:
            out.append("\\u%04x" % c)
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def dump(obj) -> str:
    """nlohmann::json::dump() of a JSON value given as Python objects (floats stay floats)."""
    if obj is None:
        return "null"
    if obj is True:
        return "true"
    if obj is False:
        return "false"
    if isinstance(obj, int):
        return str(obj)
    if isinstance(obj, float):
        return fmt_double(obj)
    if isinstance(obj, str):
        return _quote(obj)
    if isinstance(obj, (list, tuple)):
        return "[" + ",".join(dump(x) for x in obj) + "]"
    if isinstance(obj, dict):
        return "{" + ",".join(_quote(k) + ":" + dump(obj[k]) for k in sorted(obj)) + "}"
    raise TypeError(type(obj))
