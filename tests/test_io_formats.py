"""The reference's on-disk formats through the C ABI (host code, no GPU):
unisparse.tn tensors (tensor_io.cpp:31-81; test_core.cpp:122-171) and the RLE
block-mask JSON (selection.cpp:90-144; test_selection.cpp:142-172), the latter
checked byte for byte against nlohmann::json — the serializer the reference
uses — compiled from the copy vendored in this image."""
import os
import subprocess

import numpy as np
import pytest

from paper_2512_14082_b200 import api

NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"


def test_tensor_round_trips_bit_exactly(tmp_path):  # test_core.cpp:122-136
    rng = np.random.default_rng(7)
    x = rng.standard_normal((3, 64, 16)).astype(np.float32)
    x[0, 0, 0] = np.float32(-0.0)
    x[1, 2, 3] = np.float32(np.inf)
    p = str(tmp_path / "t.bin")
    api.write_tensor(p, x)
    y = api.read_tensor(p)
    assert y.shape == (3, 64, 16)
    assert (y.view(np.uint32) == x.view(np.uint32)).all()
    assert os.path.getsize(p) == 16 + 12 + 4 * 3 * 64 * 16
    raw = open(p, "rb").read()
    assert raw[:12] == b"unisparse.tn" and np.frombuffer(raw[12:28], "<u4").tolist() == [1, 3, 64, 16]


def test_tensor_reader_rejects_malformed_files(tmp_path):  # test_core.cpp:138-171
    ok = str(tmp_path / "ok.bin")
    api.write_tensor(ok, np.ones((1, 32, 8), np.float32))
    bad = tmp_path / "bad_magic.bin"
    bad.write_bytes(b"wrongmagic!!" + bytes(100))
    with pytest.raises(api.IoError, match="bad magic at offset 0"):
        api.read_tensor(str(bad))
    short = tmp_path / "short.bin"
    short.write_bytes(open(ok, "rb").read()[:-16])
    with pytest.raises(api.IoError, match="payload shorter than header"):
        api.read_tensor(str(short))
    long = tmp_path / "long.bin"
    long.write_bytes(open(ok, "rb").read() + b"extra")
    with pytest.raises(api.IoError, match="trailing bytes"):
        api.read_tensor(str(long))
    ver = tmp_path / "ver.bin"
    b = bytearray(open(ok, "rb").read())
    b[12] = 2
    ver.write_bytes(bytes(b))
    with pytest.raises(api.IoError, match="unsupported version 2 at offset 12"):
        api.read_tensor(str(ver))
    with pytest.raises(api.IoError):
        api.read_tensor(str(tmp_path / "nope.bin"))


def _bits(mask):
    P_, N, _ = mask.shape
    W = (N + 31) // 32
    pad = np.zeros((P_, N, W * 32), bool)
    pad[..., :N] = mask
    return (pad.reshape(P_, N, W, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)).sum(-1).astype(np.uint32)


def test_mask_json_round_trips(tmp_path):  # test_selection.cpp:142-153
    rng = np.random.default_rng(13)
    N = 40
    m = (rng.random((2, N, N)) < 0.3) & np.tril(np.ones((N, N), bool))
    p = str(tmp_path / "mask.json")
    api.save_mask_json_bits(p, _bits(m), 2, N, 1, 0.85)
    r, P = api.load_mask_json(p)
    assert P == 0.85 and (r == m).all()
    # head broadcast (c_h = 2): one plane, two heads
    api.save_mask_json_bits(p, _bits(m[:1]), 2, N, 2, 0.85)
    r, _ = api.load_mask_json(p)
    assert (r[0] == m[0]).all() and (r[1] == m[0]).all()


def test_mask_json_runs_kat(tmp_path):  # test_selection.cpp:155-172
    plane = np.zeros((1, 4, 4), bool)
    plane[0, 3, [0, 1, 3]] = True
    plane[0, [0, 1, 2], [0, 1, 2]] = True
    p = str(tmp_path / "runs.json")
    api.save_mask_json_bits(p, _bits(plane), 1, 4, 1, 0.5)
    r, _ = api.load_mask_json(p)
    assert (r == plane).all() and r[0, 3].sum() == 3
    assert '\t\t\t\t[0,2],\n\t\t\t\t[3,1]\n' in open(p).read()  # runs of row 3


NLOHMANN_PROG = r"""
#include <fstream>
#include <iostream>
#include <nlohmann/json.hpp>
// the reference's save_mask_json (selection.cpp:90-117) on a mask read from stdin:
// H N P, then H*N rows of N 0/1 digits
int main(int argc, char** argv) {
  int H, N; double P;
  std::cin >> H >> N >> P;
  nlohmann::json j;
  j["version"] = 1; j["H"] = H; j["N"] = N; j["P"] = P;
  auto& heads = j["heads"] = nlohmann::json::array();
  for (int h = 0; h < H; ++h) {
    nlohmann::json rows = nlohmann::json::array();
    for (int i = 0; i < N; ++i) {
      std::string bits; std::cin >> bits;
      nlohmann::json runs = nlohmann::json::array();
      int j0 = -1;
      for (int b = 0; b <= N; ++b) {
        const bool on = b < N && bits[b] == '1';
        if (on && j0 < 0) j0 = b;
        if (!on && j0 >= 0) { runs.push_back({j0, b - j0}); j0 = -1; }
      }
      rows.push_back(std::move(runs));
    }
    heads.push_back(std::move(rows));
  }
  std::ofstream os(argv[1]);
  os << j.dump(1, '\t') << "\n";
}
"""


@pytest.mark.skipif(not os.path.exists(os.path.join(NLOHMANN, "nlohmann", "json.hpp")),
                    reason="nlohmann/json.hpp not vendored in this image")
@pytest.mark.parametrize("P", [0.95, 0.9, 1.0, 0.5])
def test_mask_json_bytes_equal_nlohmann(tmp_path, P):
    src = tmp_path / "ref_save.cpp"
    src.write_text(NLOHMANN_PROG)
    exe = tmp_path / "ref_save"
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-O1", "-std=c++17", f"-I{NLOHMANN}", str(src), "-o", str(exe)], check=True)
    rng = np.random.default_rng(int(P * 100))
    H, N = 3, 37
    m = (rng.random((H, N, N)) < 0.35) & np.tril(np.ones((N, N), bool))
    m[1, 5] = False  # an empty row -> []
    stdin = f"{H} {N} {P!r}\n" + "\n".join("".join("1" if v else "0" for v in m[h, i])
                                            for h in range(H) for i in range(N)) + "\n"
    ref = tmp_path / "ref.json"
    subprocess.run([str(exe), str(ref)], input=stdin, text=True, check=True)
    ours = tmp_path / "ours.json"
    api.save_mask_json_bits(str(ours), _bits(m), H, N, 1, P)
    assert ours.read_bytes() == ref.read_bytes()


def test_metrics_csv_format(tmp_path):
    """write_metrics_csv (experiment.cpp:129-142): header and %.9g numbers."""
    from paper_2512_14082_b200 import experiment as E
    r = E.RunRow(proxy=1, c_q=8, c_k=8, c_h=2, strategy=2, P=0.95, causal_mode=0, rho=0.123456789012,
                 spearman=1.0, recall=2.0 / 3.0, max_abs=1e-10, cosine=0.999999999999, selection_flops=12,
                 attention_flops=3 * 2 ** 40)
    E.write_metrics_csv([r], str(tmp_path / "m.csv"))
    lines = (tmp_path / "m.csv").read_text().splitlines()
    assert lines[0] == "proxy,c_q,c_k,c_h,strategy,P,rho,spearman,recall,max_abs,cosine,selection_flops,attention_flops"
    assert lines[1] == "antidiagonal,8,8,2,stochastic,0.95,0.123456789,1,0.666666667,1e-10,1,12,3298534883328"
