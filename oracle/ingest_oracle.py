"""CPU restatement of the dataset side of the path.

TEST INFRASTRUCTURE ONLY: imported by tests/ as a checker, never by the
product.  Pure Python (small files only).

  load_records  <- load_record_file + load_dataset truncation
                   (/root/reference/proj/src/workload.cpp:65-103, 109-127)
  draw_all      <- run_plan's draw loop (driver.cpp:209-215) over
                   draw_minibatch (workload.cpp:129-146)

Pinned against the compiled reference on tests/ingest_cases.py
(tests/test_ingest_oracle.py)."""
from __future__ import annotations

MISSING_TAB, NOT_INTEGERS, INPUT_LT_1, TARGET_LT_0 = 0, 1, 2, 3
_WS = b" \t\n\v\f\r"
_LLMAX = (1 << 63) - 1


def _stoll_full(field: bytes):
    """std::stoll(field, &used) with used == len(field) (workload.cpp:83-88):
    leading isspace, optional sign, >= 1 digit, nothing after, int64 range."""
    k = 0
    while k < len(field) and field[k] in _WS:
        k += 1
    neg = False
    if k < len(field) and field[k] in b"+-":
        neg = field[k] == ord("-")
        k += 1
    d0 = k
    while k < len(field) and 48 <= field[k] <= 57:
        k += 1
    if k == d0 or k != len(field):
        return None
    v = int(field[d0:k])
    v = -v if neg else v
    if v > _LLMAX or v < -_LLMAX - 1:
        return None  # std::out_of_range
    return v


def load_records(data: bytes, max_seq_len: int):
    """-> ("ok", [(id, input, target)]) | ("parse", line, byte, kind) | ("invalid",)."""
    if max_seq_len < 1:
        return ("invalid",)
    out = []
    lines = data.split(b"\n")
    if data.endswith(b"\n"):
        lines = lines[:-1]  # getline: no empty line after the final newline
    off = 0
    for no, line in enumerate(lines, 1):
        start = off
        off += len(line) + 1
        if not line or line[0] == ord("#"):
            continue
        tab = line.find(b"\t")
        if tab < 0:
            return ("parse", no, start, MISSING_TAB)
        a, b = _stoll_full(line[:tab]), _stoll_full(line[tab + 1:])
        if a is None or b is None:
            return ("parse", no, start, NOT_INTEGERS)
        if a < 1:
            return ("parse", no, start, INPUT_LT_1)
        if b < 0:
            return ("parse", no, start, TARGET_LT_0)
        out.append((len(out), min(a, max_seq_len), min(b, max_seq_len)))
    if not out:
        return ("invalid",)  # "dataset is empty" (workload.cpp:121)
    return ("ok", out)


def draw_all(samples, budget: int):
    """Segment offsets of every mini-batch drawn from cursor 0."""
    if budget < 1:
        raise ValueError("token_budget must be >= 1")
    offs, cur, n = [0], 0, len(samples)
    while cur < n:
        tokens = 0
        while cur < n:
            tokens += int(samples[cur][1]) + int(samples[cur][2])
            cur += 1
            if tokens >= budget:
                break  # the crossing sample stays
        offs.append(cur)
    return offs
