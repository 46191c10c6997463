"""Command-line front end (cli.py; reference tools/geodist_main.cpp): exit codes, input
validation and the CSV / JSON formats.  GPU cases run the subcommands end to end."""
import csv
import json
import math

import numpy as np
import pytest

from conftest import bits, golden

import paper_1810_08218_b200 as g
from paper_1810_08218_b200 import cli


def test_format_distance():
    # format_distance (mesh_io.cpp): %.17g, ".0" appended to integral output, inf spelled out
    assert cli.format_distance(1.0) == "1.0"
    assert cli.format_distance(0.0) == "0.0"
    assert cli.format_distance(math.inf) == "inf"
    assert cli.format_distance(0.1) == "0.10000000000000001"
    assert cli.format_distance(1e20) == "1e+20"
    assert cli.format_distance(2.5) == "2.5"


def test_colors():
    # distance ramp contract (mesh_io.hpp): R = round(255u), G = round(255(1-|2u-1|)), B = round(255(1-u))
    assert cli.distance_color(0.0, 2.0) == (0, 0, 255)
    assert cli.distance_color(1.0, 2.0) == (128, 255, 128)
    assert cli.distance_color(math.inf, 2.0) == (255, 0, 0)
    assert cli.label_color(-1) == (128, 128, 128)
    assert all(0 <= c < 256 for c in cli.label_color(12345))


@pytest.mark.parametrize("argv", [
    [],                                                   # no subcommand
    ["geodesic", "--sphere", "2"],                        # --source required
    ["geodesic", "--grid", "4", "--source", "0"],         # NX,NY
    ["geodesic", "--grid", "1,5", "--source", "0"],       # sizes >= 2
    ["geodesic", "--grid", "4,x", "--source", "0"],       # invalid size
    ["geodesic", "--grid", "4,4,s", "--source", "0"],     # invalid shear
    ["geodesic", "--sphere", "10", "--source", "0"],      # subdivision range
    ["geodesic", "--sphere", "2", "--grid", "3,3", "--source", "0"],  # excludes
    ["geodesic", "--source", "0"],                        # one input required
    ["fps", "--sphere", "1"],                             # --count required
    ["bench", "--sphere", "1"],                           # --sources-range required
    ["geodesic", "--mesh", "/nonexistent/m.off", "--source", "0"],
])
def test_input_errors_exit_2(argv, capsys):
    assert cli.main(argv) == cli.EXIT_INPUT


@pytest.mark.gpu
def test_geodesic_end_to_end(tmp_path):
    gd = golden("ico3_src0")
    out, st, tr = tmp_path / "d.csv", tmp_path / "s.json", tmp_path / "t.csv"
    rc = cli.main(["geodesic", "--sphere", "3", "--source", "0", "--out-csv", str(out),
                   "--stats", str(st), "--trace", str(tr), "--out-ply", str(tmp_path / "d.ply")])
    assert rc == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["index", "distance", "label"]
    d = np.array([float(r[1]) for r in rows[1:]])
    assert np.array_equal(bits(d), bits(gd["dist_d"]))
    assert all(r[2] == "-1" for r in rows[1:])
    s = json.load(open(st))
    assert s["iterations"] == int(gd["K_d"]) and s["relax_calls"] == int(gd["relax_d"])
    assert s["manifest"]["command"] == "geodesic" and s["manifest"]["sources"] == [0]
    assert 0 < s["mape_percent"] < 5
    assert open(tr).readline() == "k,i,j,updated,max_rel_change\n"
    assert cli.main(["geodesic", "--sphere", "2", "--source", "99999"]) == cli.EXIT_INPUT
    assert cli.main(["geodesic", "--sphere", "2", "--source", "0", "--method", "fm"]) == cli.EXIT_INPUT


@pytest.mark.gpu
def test_fps_and_bench_end_to_end(tmp_path):
    out, st, dist = tmp_path / "f.csv", tmp_path / "f.json", tmp_path / "fd.csv"
    assert cli.main(["fps", "--grid", "20,20", "--count", "6", "--seed", "3", "--out-csv", str(out),
                     "--stats", str(st), "--out-dist", str(dist)]) == 0
    M = g.generate_grid(20, 20)
    ref = g.farthest_point_sampling(M, 6, seed=3)
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["order", "vertex", "insertion_radius"]
    assert [int(r[1]) for r in rows[1:]] == list(ref["samples"])
    assert rows[1][2] == "inf"
    s = json.load(open(st))
    assert s["samples"] == list(map(int, ref["samples"])) and len(s["iterations"]) == 6
    assert cli.main(["fps", "--grid", "4,4", "--count", "99"]) == cli.EXIT_INPUT
    b = tmp_path / "b.csv"
    assert cli.main(["bench", "--sphere", "2", "--sources-range", "1:3", "--out-csv", str(b)]) == 0
    rows = list(csv.reader(open(b)))
    assert rows[0] == ["m", "rho", "iterations", "ptp_relax_calls"] and len(rows) == 4
