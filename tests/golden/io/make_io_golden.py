"""Golden data for the file-format cross-checks (run in the build container,
where /root/reference exists; oracle/Makefile builds oracle/_ref/ref_io
from the unmodified reference io.hpp).

  tests/golden/io/ref/*     the fixed objects of objects.hpp, written by the
                            reference formatters
  tests/golden/io/cases.tsv <kind> <reference outcome> <base64 document>: valid
                            documents and deterministic corruptions of them,
                            with the reference parser's outcome ("ok" or the
                            errc ordinal) -- tests/cpp/test_io.cpp requires
                            the same outcome from include/tsdict/io.hpp
usage: python tests/golden/io/make_io_golden.py"""
import base64
import os
import random
import struct
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(HERE)))
REF_IO = os.path.join(ROOT, "oracle", "_ref", "ref_io")


def explicit_cases():
    """hand-written edge cases (the behaviours the reference's test_io.cpp names, and more)"""
    c = []
    s = lambda d: c.append(("series", d.encode() if isinstance(d, str) else d))
    for d in ["# n=3\n1\n2\n3\n", "1\n2\n3\n", "# n=2\r\n1.5\r\n2.5\r\n", "# n=4\n1\n2\n3\n", "1\n# n=2\n2\n",
              "# comment\n1\n", "# n=two\n1\n", "", "   \n\n", "# n=0\n", "1\nabc\n2\n", "1\n2.5.3\n", "1\ninf\n",
              "nan\n", "-inf\n", "1e308\n", "1e309\n", "0x10\n", "+1\n", " 1 \n 2\n", "1\n\n2\n", "1 2\n", "#n=1\n1\n",
              "# n=1\n1", "1e-320\n", ".5\n", "5.\n", "-0\n", "# n= 2\n1\n2\n", "# n=2 \n1\n2\n"]:
        s(d)
    good = b"MPD1" + struct.pack("<Q", 3) + struct.pack("<3d", 1.0, 2.0, 3.0)
    s(good)
    s(good[:-1])
    s(good[:8])
    s(good[:4])
    s(b"MPD1" + struct.pack("<Q", 4) + good[12:])
    s(b"MPD1" + struct.pack("<Q", 1 << 61))
    s(b"MPD1" + struct.pack("<Q", 0))
    s(good[:20] + struct.pack("<d", float("nan")) + good[28:])
    s(good[:12] + struct.pack("<d", float("inf")) + good[20:])
    s(b"MPD2" + good[4:])
    s(good + b"\x00")
    p = lambda d: c.append(("profile", d.encode()))
    base = "# m=4 kind=ab-join\nwindow_start\tdistance\tnn_index\n"
    for d in ["", "window_start\tdistance\tnn_index\n0\t1\t2\n", "# m=10 kind=self-join\n",
              "# m=10 kind=sideways\nwindow_start\tdistance\tnn_index\n",
              "# m=1 kind=self-join\nwindow_start\tdistance\tnn_index\n",
              "# m=10 kind=self-join\nwindow_start\tdistance\tnn_index\n", base + "0\t0.5\t3\n", base + "1\t0.5\t3\n",
              base + "0\t0.5\t3\n2\t0.5\t3\n", base + "0\t-0.5\t3\n", base + "0\tnan\t3\n", base + "0\t0.5\t-2\n",
              base + "0\t0.5\n", base + "0\t0.5\tthree\n", base + "0\tinf\t-1\n", base + "0\t0.5\t3\t4\n",
              "# m=4\nwindow_start\tdistance\tnn_index\n0\t1\t2\n", "# kind=ab-join\nwindow_start\tdistance\tnn_index\n0\t1\t2\n",
              "# m=x kind=ab-join\nwindow_start\tdistance\tnn_index\n0\t1\t2\n",
              base.replace("nn_index", "neighbor") + "0\t1\t2\n", base + "0 0.5 3\n", base + "0\t0.5\t3\r\n"]:
        p(d)
    l = lambda d: c.append(("labels", d.encode()))
    for d in ["# start\tend\n10\t50\n40\t90\n", "5\t10\n20\t30\n", "", "# only a comment\n", "5\t5\n", "6\t5\n",
              "1\t2\t3\n", "a\tb\n", "-1\t5\n", "1 2\n", "3\t9", "0\t18446744073709551615\n", "\n\n1\t2\n\n"]:
        l(d)
    d = lambda t: c.append(("dictionary", t.encode()))
    for t in ["not json at all {{{", "[1,2,3]", "", "{}", "null", "{\"format_version\":1}", "{\"format_version\":2}",
              "{\"format_version\":\"1\"}", "{\"format_version\":1.0}", "{\"format_version\":1", "{\"a\":1,}", "[", "\"x\"",
              "{\"format_version\":1,\"m\":16,\"k\":1.5,\"source_length\":100,\"space_saving\":0.5,\"e_max\":null,"
              "\"core_starts\":[],\"segments\":[{\"start\":0,\"length\":50,\"values\":[" + ",".join(["1"] * 50) + "]}]}"]:
        d(t)
    return c


def corruptions(kind, doc, rng, n):
    out = []
    text = doc.decode("latin-1")
    for _ in range(n):
        op = rng.randrange(7)
        if op == 0 and len(doc) > 1:  # truncate
            out.append(doc[: rng.randrange(1, len(doc))])
        elif op == 1:  # replace one byte
            i = rng.randrange(len(doc))
            out.append(doc[:i] + bytes([rng.choice(b"0123456789.-+eE,:[]{}\"\t\n #xnal")]) + doc[i + 1:])
        elif op == 2:  # delete one byte
            i = rng.randrange(len(doc))
            out.append(doc[:i] + doc[i + 1:])
        elif op == 3 and "\n" in text:  # drop a line
            lines = text.split("\n")
            del lines[rng.randrange(len(lines))]
            out.append("\n".join(lines).encode("latin-1"))
        elif op == 4 and "\n" in text:  # duplicate a line
            lines = text.split("\n")
            i = rng.randrange(len(lines))
            lines.insert(i, lines[i])
            out.append("\n".join(lines).encode("latin-1"))
        elif op == 5:  # swap two bytes
            i, j = sorted(rng.sample(range(len(doc)), 2))
            b = bytearray(doc)
            b[i], b[j] = b[j], b[i]
            out.append(bytes(b))
        else:  # insert a byte
            i = rng.randrange(len(doc) + 1)
            out.append(doc[:i] + bytes([rng.choice(b"0123456789.-e,\"\t\n ")]) + doc[i:])
    return [(kind, o) for o in out]


def json_edits(doc, rng):
    """structural edits of a valid dictionary document (keys, types, values)"""
    import json
    base = json.loads(doc)
    out = []

    def emit(j):
        out.append(("dictionary", json.dumps(j, separators=(",", ":")).encode()))

    for key in list(base.keys()):
        j = dict(base); del j[key]; emit(j)  # missing key
        for v in (None, "x", -1, 0, 2, 1.5, [], 2 ** 64 - 1):
            j = dict(base); j[key] = v; emit(j)
    j = dict(base); j["future_field"] = 1; emit(j)
    for sk in ("start", "length", "values"):
        for v in (None, "x", 15, 16, 2 ** 64 - 1, [1.0]):
            j = json.loads(doc); j["segments"][0][sk] = v; emit(j)
        j = json.loads(doc); del j["segments"][0][sk]; emit(j)
    j = json.loads(doc); j["segments"][1]["note"] = "x"; emit(j)
    j = json.loads(doc); j["segments"][1]["start"] = j["segments"][0]["start"]; emit(j)
    j = json.loads(doc); j["segments"].reverse(); emit(j)
    j = json.loads(doc); j["segments"] = []; emit(j)
    j = json.loads(doc); j["segments"][0]["values"][3] = "nan"; emit(j)
    j = json.loads(doc); j["space_saving"] += 1e-13; emit(j)
    j = json.loads(doc); j["space_saving"] += 1e-11; emit(j)
    for cs in ([], [0], [984], [985], [999], [1000], [10, 18], [10, 19], [19, 10], [10, 10], [-1]):  # m = 16
        j = json.loads(doc); j["core_starts"] = cs; emit(j)
    for k in (0.0, -1.5, 0.5):
        j = json.loads(doc); j["k"] = k; emit(j)
    return out


def main():
    # --fuzz N DIR: a larger throw-away set (N corruptions per file, another
    # seed) into DIR instead of the committed golden data
    import sys
    fuzz = "--fuzz" in sys.argv
    per_file = int(sys.argv[sys.argv.index("--fuzz") + 1]) if fuzz else 40
    out_dir = sys.argv[sys.argv.index("--fuzz") + 2] if fuzz else HERE
    os.makedirs(os.path.join(out_dir, "ref"), exist_ok=True)
    subprocess.run([REF_IO, "write", os.path.join(out_dir, "ref")], check=True)
    rng = random.Random(7 if fuzz else 20261020)
    cases = explicit_cases()
    files = {"series": ["series.txt", "series.mpd1"], "dictionary": ["dict.json", "dict_null_emax.json"],
             "profile": ["profile_self.tsv", "profile_ab.tsv"], "labels": ["labels.tsv"]}
    for kind, names in files.items():
        for name in names:
            with open(os.path.join(out_dir, "ref", name), "rb") as f:
                doc = f.read()
            cases.append((kind, doc))
            cases += corruptions(kind, doc, rng, per_file)
    with open(os.path.join(out_dir, "ref", "dict.json"), "rb") as f:
        cases += json_edits(f.read().decode(), rng)
    inp = "".join(f"{k}\t{d.hex()}\n" for k, d in cases)  # the driver reads hex
    r = subprocess.run([REF_IO, "codes"], input=inp, capture_output=True, text=True, check=True)
    outcomes = r.stdout.split()
    assert len(outcomes) == len(cases)
    with open(os.path.join(out_dir, "cases.tsv"), "w") as f:
        for (k, d), o in zip(cases, outcomes):
            f.write(f"{k}\t{o}\t{base64.b64encode(d).decode()}\n")
    print(len(cases), "cases;", sum(o == "ok" for o in outcomes), "accepted")


if __name__ == "__main__":
    main()
