"""Monte-Carlo report rows and sweep bookkeeping, on CPU:
the CSV row is byte-identical to the reference's format_csv_row (its own
known-answer row, test_sim.cpp:175-223, and the compiled reference on random
statistics); the sweep enumerates and validates like run_montecarlo."""
import io

import numpy as np
import pytest

KAT = ("2.25,10240,12345,678,1.177311e-03,6.621094e-02,123.457,89.012,"
       "456.789,1.5000")


@pytest.fixture(scope="module")
def S(native):
    from paper_1710_08314_b200 import sim

    return sim


def _kat(S):
    return S.PointStats(2.25, 10240, 12345, 678, 12345 / (1024.0 * 10240.0), 678 / 10240.0,
                        123.4567, 89.0123, 456.789, 1.5)


def test_csv_row_known_answer(S):
    assert S.format_csv_row(_kat(S)) == KAT


def test_report_csv_and_table(S):
    buf = io.StringIO()
    S.write_report(buf, "csv", ["seed: 42", "decoder: SSC"], [_kat(S)])
    text = buf.getvalue()
    assert "# seed: 42\n" in text and "# decoder: SSC\n" in text
    assert ("ebn0_db,frames,bit_errors,frame_errors,ber,fer,ti_mbps,lat_avg_us,lat_worst_us,"
            "esc_mean\n") in text
    assert KAT + "\n" in text
    # numeric round trip of the row
    v = [float(x) for x in KAT.split(",")]
    assert v[0] == 2.25 and int(v[1]) == 10240 and int(v[2]) == 12345 and int(v[3]) == 678
    tab = io.StringIO()
    S.write_report(tab, "table", ["seed: 42"], [_kat(S)])
    lines = tab.getvalue().splitlines()
    assert lines[0] == "# seed: 42" and "ebn0_db" in lines[1] and "2.25" in lines[2]
    assert len(lines[1]) == len(lines[2])  # column-aligned


def test_csv_row_matches_compiled_reference(S, ref_lib):
    from oracle.oracle import ref_format_csv_row

    rng = np.random.default_rng(3)
    for _ in range(200):
        fr = int(rng.integers(1, 10**9))
        fe = int(rng.integers(0, fr + 1))
        be = int(rng.integers(fe, 50 * fe + 1))
        p = S.PointStats(float(rng.choice([0.25, 1.0, 2.5, -1.5, 3.3333333333, 10.0])), fr, be, fe,
                         be / (fr * 1723.0), fe / fr, float(rng.uniform(0, 1e5)),
                         float(rng.uniform(0, 1e4)), float(rng.uniform(0, 1e5)),
                         float(rng.uniform(1, 32)))
        vals = [p.ebn0_db, p.frames, p.bit_errors, p.frame_errors, p.ber, p.fer, p.ti_mbps,
                p.lat_avg_us, p.lat_worst_us, p.esc_mean]
        assert S.format_csv_row(p) == ref_format_csv_row(vals)


def test_sweep_points_and_validation(S, native):
    import paper_1710_08314_b200 as P

    code = P.make_code(16, 8, P.construct_frozen(16, 8, 0.5))
    cfg = S.SimConfig(code, ebn0_min=1.0, ebn0_max=4.0, ebn0_step=0.5)
    assert list(S.points(cfg)) == [1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0]
    cfg = S.SimConfig(code, ebn0_min=0.0, ebn0_max=0.3, ebn0_step=0.1)
    assert len(list(S.points(cfg))) == 4  # the 1e-9 slack of sim.cpp:141
    for bad in (dict(ebn0_step=0), dict(ebn0_min=2, ebn0_max=1), dict(max_frames=0, max_fe=0),
                dict(channel="x")):
        with pytest.raises(P.ConfigError):
            S._validate(S.SimConfig(code, **bad))
