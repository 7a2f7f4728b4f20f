"""Host-side logic of the drop-in API (no GPU): validation messages, grids,
Karmarkar-Karp scheduling, cost model, I/O, evaluation and the contract helpers.
Examples follow the reference's own tests (pkg/tests/test_*.py)."""

from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2401_13680_b200 as P


class TestSeriesValidation:
    def test_readonly_and_dtype(self):
        s = P.TimeSeries([1.0, 2.0, 3.0])
        assert s.n == 3 and s.values.dtype == np.float64
        with pytest.raises(ValueError):
            s.values[0] = 9.0

    def test_errors(self):
        with pytest.raises(ValueError, match="one-dimensional"):
            P.TimeSeries(np.ones((2, 2)))
        with pytest.raises(ValueError, match="at least 2"):
            P.TimeSeries([1.0])
        with pytest.raises(ValueError, match="position 2"):
            P.TimeSeries([1.0, 2.0, np.nan, 4.0])
        with pytest.raises(ValueError, match="position 0"):
            P.TimeSeries([np.inf, 2.0])

    def test_scaled(self):
        out = P.TimeSeries([1.0, -2.0], coordinate_id=3).scaled(2.5)
        np.testing.assert_allclose(out.values, [2.5, -5.0])
        assert out.coordinate_id == 3


class TestIO:
    def test_roundtrip_and_header(self, tmp_path):
        rng = np.random.default_rng(7)
        s = P.TimeSeries(rng.standard_normal(50) * 1e3)
        p = tmp_path / "s.csv"
        P.save_series(s, p)
        np.testing.assert_array_equal(P.load_series(p).values, s.values)
        p.write_text("value\n1.0\n2.0\n")
        np.testing.assert_array_equal(P.load_series(p).values, [1.0, 2.0])

    def test_bad_cells(self, tmp_path):
        p = tmp_path / "s.csv"
        p.write_text("1.0\n2.0\n3.0\n4.0\nabc\n6.0\n")
        with pytest.raises(ValueError, match="row 5"):
            P.load_series(p)
        with pytest.raises(FileNotFoundError):
            P.load_series(tmp_path / "nope.csv")
        p.write_text("1.0,10.0\n2.0,20.0\n")
        assert P.load_series(p, column=1).coordinate_id == 1
        with pytest.raises(ValueError, match="column"):
            P.load_series(p, column=4)

    def test_labels_io(self, tmp_path):
        lab = P.LabelSequence(np.array([0, 1, 1, 0]))
        p = tmp_path / "l.txt"
        P.write_labels(lab, p)
        np.testing.assert_array_equal(P.read_labels(p).labels, lab.labels)


class TestParams:
    def test_defaults(self):
        assert [P.default_window_size(m) for m in (32, 7, 2)] == [16, 4, 1]
        assert [P.default_order_stat(m) for m in (32, 8, 100, 2)] == [4, 1, 10, 1]
        p = P.MPdistParams(32)
        assert (p.window_size, p.k, p.profile_width) == (16, 4, 17)

    def test_errors(self):
        with pytest.raises(ValueError, match="window size"):
            P.MPdistParams(8, window_size=9)
        with pytest.raises(ValueError, match="snippet size"):
            P.MPdistParams(1)
        with pytest.raises(ValueError, match="order statistic"):
            P.MPdistParams(8, k=0)

    def test_integer_defaults_match_float_formulas(self):
        import math
        for m in range(2, 20000, 7):
            assert P.default_order_stat(m) == max(1, -(-m // 10)) == max(1, math.ceil(0.05 * 2 * m))


class TestHelpers:
    def test_column_minima(self):
        np.testing.assert_array_equal(P.column_minima([[1.0, 4.0, 2.0], [3.0, 0.0, 5.0]]), [1.0, 0.0, 2.0])
        with pytest.raises(ValueError, match="length"):
            P.column_minima([np.array([1.0, 2.0]), np.array([1.0])])

    def test_row_sliding_minima(self):
        np.testing.assert_array_equal(P.row_sliding_minima([3.0, 1.0, 2.0, 5.0, 4.0], 2), [1.0, 1.0, 2.0, 4.0])
        with pytest.raises(ValueError, match="window"):
            P.row_sliding_minima([1.0, 2.0], 3)

    @given(st.lists(st.floats(min_value=-1e6, max_value=1e6, allow_nan=False), min_size=1, max_size=80), st.data())
    @settings(max_examples=80, deadline=None)
    def test_sliding_minima_brute(self, row, data):
        w = data.draw(st.integers(min_value=1, max_value=len(row)))
        brute = np.array([min(row[j:j + w]) for j in range(len(row) - w + 1)])
        np.testing.assert_array_equal(P.row_sliding_minima(row, w), brute)

    def test_mpdist_at(self):
        p = P.MPdistParams(3, window_size=2, k=1)
        assert P.mpdist_at([0.1, 0.4], [0.2, 0.3], p) == pytest.approx(0.1)
        p9 = P.MPdistParams(3, window_size=2, k=9)
        assert P.mpdist_at([0.1, 0.4], [0.2, 0.3], p9) == pytest.approx(0.4)
        with pytest.raises(ValueError, match="halves"):
            P.mpdist_at([0.1], [0.2, 0.3], p)

    def test_curve_area(self):
        np.testing.assert_array_equal(P.representativeness_curve([[1.0, 3.0, 2.0], [2.0, 1.0, 4.0]]),
                                      [1.0, 1.0, 2.0])
        assert P.profile_area([1.0, 1.0, 2.0]) == 4.0
        with pytest.raises(ValueError, match="non-empty"):
            P.representativeness_curve([])

    def test_segment(self):
        np.testing.assert_array_equal(P.segment(P.TimeSeries(np.arange(9.0)), 2).starts, [0, 2, 4, 6])
        with pytest.raises(ValueError, match="at least 2"):
            P.segment(P.TimeSeries(np.arange(9.0)), 5)

    def test_znorm_distance(self):
        assert P.znorm_distance([1.0, 2.0, 3.0], [3.0, 2.0, 1.0]) == pytest.approx(2 * np.sqrt(3))
        assert P.znorm_distance([4.0, 4.0], [9.0, 9.0]) == 0.0
        assert P.znorm_distance([7.0] * 4, [0.0, 1.0, 2.0, 3.0]) == pytest.approx(2.0)


class TestLengthSelectHost:
    def test_make_grid(self):
        assert P.make_grid(8, 64) == [8, 16, 32, 64]
        assert P.make_grid(8, 63) == [8, 16, 32]
        assert P.make_grid(10, 30, rule="arith", step=10) == [10, 20, 30]
        with pytest.raises(ValueError, match="smaller than m_min"):
            P.make_grid(16, 8)
        with pytest.raises(ValueError, match="grid rule"):
            P.make_grid(4, 8, rule="geom")
        with pytest.raises(ValueError, match="step"):
            P.make_grid(4, 8, rule="arith", step=0)

    def test_select_length_arg_errors(self):
        s = P.TimeSeries(np.arange(64.0))
        with pytest.raises(ValueError, match="empty"):
            P.select_length(s, [], 2)
        with pytest.raises(ValueError, match="duplicates"):
            P.select_length(s, [8, 8], 2)
        with pytest.raises(ValueError, match="at least 2"):
            P.select_length(s, [8], 1)

    def test_criterion_errors(self):
        res = P.SnippetResult(4, 2, 1, 5, (), np.zeros(2), 0.0,
                              (P.MPdistProfile(0, np.array([0.0, 2.0])),), 2.0, np.zeros(1, dtype=np.int64), 0)
        with pytest.raises(ValueError, match="at least 2"):
            P.criterion_score(res)


class TestScheduler:
    def test_kk_example(self):
        sched = P.kk_partition([7, 5, 4, 8, 6], 2)
        sets = sorted(sorted([7, 5, 4, 8, 6][i] for i in part) for part in sched.assignments)
        assert sets == [[4, 5, 7], [6, 8]]
        assert sched.difference == Fraction(2)

    @given(st.lists(st.floats(min_value=0.1, max_value=100.0), min_size=1, max_size=20),
           st.integers(min_value=1, max_value=5))
    @settings(max_examples=60, deadline=None)
    def test_kk_partition_exact(self, weights, parts):
        sched = P.kk_partition(weights, parts)
        flat = sorted(i for a in sched.assignments for i in a)
        assert flat == list(range(len(weights)))
        loads = [sum((Fraction(weights[i]) for i in a), Fraction(0)) for a in sched.assignments]
        assert max(loads) - min(loads) == sched.difference

    def test_lpt_and_errors(self):
        assert P.lpt_partition([5, 4, 3], 2).makespan == 7.0
        with pytest.raises(ValueError, match="negative"):
            P.kk_partition([1, -1], 2)
        with pytest.raises(ValueError, match="no weights"):
            P.kk_partition([], 2)

    def test_default_cost_is_pair_count(self):
        # (m-l+1) * (n-l+1) * (n//m)
        assert P.default_cost(1000, 64) == 33 * (1000 - 32 + 1) * (1000 // 64)

    def test_cost_model(self, tmp_path):
        m = np.array([8, 16, 32, 64.0])
        model = P.fit_cost_model(m, 0.5 + 0.01 * m ** 2)
        assert model.degree == 2
        assert model.predict(32) == pytest.approx(0.5 + 0.01 * 32 ** 2)
        with pytest.raises(ValueError, match="distinct"):
            P.fit_cost_model([8, 8, 8], [1, 2, 3])
        log = tmp_path / "t.jsonl"
        log.write_text('{"m": 8, "n": 100, "l": 4, "seconds": 1.5, "timestamp": "x"}\n'
                       '{"m": 16, "n": 200, "l": 8, "seconds": 2.5, "timestamp": "x"}\n')
        ms, secs = P.load_training_samples(log, series_length=100)
        assert list(ms) == [8.0] and list(secs) == [1.5]

    def test_run_schedule_errors(self):
        s = P.TimeSeries(np.arange(64.0))
        with pytest.raises(ValueError, match="no jobs"):
            P.run_schedule(s, [], 2)
        with pytest.raises(ValueError, match="duplicate"):
            P.run_schedule(s, [P.MPdistParams(8), P.MPdistParams(8)], 2)
        with pytest.raises(ValueError, match="at least one worker"):
            P.run_schedule(s, [P.MPdistParams(8)], 2, workers=0)


class TestEvaluate:
    def test_perfect_and_counts(self):
        t = P.LabelSequence(np.array([0, 0, 1, 1, 2, 2]))
        assert P.evaluate(t, t).macro_f1 == 1.0
        truth = P.LabelSequence(np.array([0] * 10 + [1] * 4))
        pred = P.LabelSequence(np.array([0] * 8 + [1] * 2 + [0] * 2 + [1] * 2))
        c0 = P.evaluate(pred, truth).classes[0]
        assert (c0.tp, c0.fp, c0.fn) == (8, 2, 2)

    def test_label_sequence_errors(self):
        with pytest.raises(ValueError, match="integers"):
            P.LabelSequence(np.array([0.0, 1.0]))
        with pytest.raises(ValueError, match="non-empty"):
            P.LabelSequence(np.array([], dtype=np.int64))
