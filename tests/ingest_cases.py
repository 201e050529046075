"""Record files for the dataset ingest: the reference's
load_record_file (proj/src/workload.cpp:65-103) semantics at their edges —
comments, empty lines, a last line without newline, std::stoll field rules
(leading whitespace, signs, nothing after the digits, int64 range), each
ParseError kind, lines longer than the device's 32 KB chunks — and large
seeded files."""
from __future__ import annotations

import numpy as np

EDGE = {
    "basic": b"5\t2\n9000\t1\n",
    "comments_and_blank": b"# header\n\n5\t2\n#5\t2\n\n\n7\t0\n",
    "no_trailing_newline": b"5\t2\n6\t3",
    "leading_space_and_plus": b" 5\t+2\n\t\n",
    "leading_space_both": b"  12\t  7\n+3\t 0\n",
    "crlf": b"5\t2\r\n6\t1\r\n",
    "trailing_space": b"5 \t2\n",
    "extra_tab": b"5\t2\t1\n",
    "empty_field": b"\t2\n",
    "empty_target": b"5\t\n",
    "zero_input": b"0\t3\n",
    "neg_input": b"-4\t3\n",
    "neg_target": b"4\t-1\n",
    "minus_zero_target": b"4\t-0\n",
    "missing_tab": b"5 2\n",
    "letters": b"5\t2\nnot_a_number\t1\n",
    "hex": b"0x10\t1\n",
    "llong_max": b"9223372036854775807\t9223372036854775807\n",
    "overflow": b"9223372036854775808\t1\n",
    "llong_min_target": b"5\t-9223372036854775808\n",
    "target_overflow_neg": b"5\t-9223372036854775809\n",
    "space_only_line": b" \n",
    "hash_not_first": b" #x\t1\n",
    "nul_byte": b"5\x00\t2\n",
    "only_comments": b"# a\n# b\n",
    "empty": b"",
    "newline_only": b"\n\n\n",
    "sign_only": b"+\t1\n",
    "vertical_tab_ws": b"\x0b\x0c5\t\r2\n",
    "error_after_many": b"".join(b"%d\t%d\n" % (k + 1, k % 7) for k in range(5000)) + b"3\tx\n",
}


def long_line_case():
    # a record whose leading whitespace spans several 32 KB chunks
    return b"1\t1\n" + b" " * 100_000 + b"42\t7\n" + b"3\t3"


def random_file(n, seed=5, noise=True, max_len=70000):
    rng = np.random.default_rng(seed)
    inp = np.minimum(rng.lognormal(5.0, 1.5, n).astype(np.int64) + 1, max_len)
    tgt = np.minimum(rng.lognormal(3.5, 1.2, n).astype(np.int64), max_len)
    lines = [b"%d\t%d" % (a, b) for a, b in zip(inp, tgt)]
    if noise:
        for k in rng.choice(n, size=max(1, n // 50), replace=False):
            lines[k] = [b"# comment", b"", b"  %d\t%d" % (inp[k], tgt[k]), b"+%d\t+%d" % (inp[k], tgt[k])][k % 4]
    return b"\n".join(lines) + b"\n"
