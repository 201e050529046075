"""CPU: the ingest restatement (oracle/ingest_oracle.py) pinned against the
compiled reference's load_dataset / draw_minibatch on every edge file."""
import numpy as np
import pytest

from ingest_cases import EDGE, long_line_case, random_file
from oracle import ingest_oracle as O
from oracle.bind import Reference, reference_available

pytestmark = pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("name", sorted(EDGE) + ["long_line", "random"])
def test_restatement_matches_reference(tmp_path, name):
    data = EDGE.get(name) or (long_line_case() if name == "long_line" else random_file(3000, seed=2))
    path = tmp_path / "f.tsv"
    path.write_bytes(data)
    for max_len in (8192, 3):
        rc, samples, line, byte, kind = Reference().load_record_file(str(path), max_len, cap=len(data) + 1)
        got = O.load_records(data, max_len)
        if rc == 0:
            assert got[0] == "ok" and np.array_equal(np.array(got[1], np.int64).reshape(-1, 3), samples), name
            for budget in (1, 100, 5000):
                assert O.draw_all(got[1], budget) == list(Reference().draw_all(samples, budget)[1]), name
        elif rc == 9:
            assert got == ("parse", line, byte, kind), (name, got, line, byte, kind)
        else:
            assert got == ("invalid",), name
