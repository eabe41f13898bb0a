// Host compile of the device scene builder's arithmetic (ss_build.cuh):
// reads n 3x3 matrices (row-major doubles) and n 3-vectors from stdin-named
// files, writes inverse, det and norm so tests/test_builder_math.py can
// compare them with numpy bit for bit on the CPU.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1904_02833_b200/csrc/ss_build.cuh"

int main(int argc, char** argv) {
  if (argc != 5) {
    fprintf(stderr, "usage: build_check D.bin V.bin out_inv_det.bin out_norm.bin\n");
    return 2;
  }
  auto slurp = [](const char* f) {
    std::vector<double> v;
    FILE* fp = fopen(f, "rb");
    if (!fp) return v;
    fseek(fp, 0, SEEK_END);
    v.resize(ftell(fp) / 8);
    fseek(fp, 0, SEEK_SET);
    if (fread(v.data(), 8, v.size(), fp) != v.size()) v.clear();
    fclose(fp);
    return v;
  };
  std::vector<double> D = slurp(argv[1]), V = slurp(argv[2]);
  const size_t n = D.size() / 9, m = V.size() / 3;
  std::vector<double> out(10 * n), nrm(m);
  for (size_t e = 0; e < n; ++e) out[10 * e + 9] = ssb_inv_det3(&D[9 * e], &out[10 * e]);
  for (size_t e = 0; e < m; ++e) nrm[e] = ssb_norm3(V[3 * e], V[3 * e + 1], V[3 * e + 2]);
  FILE* fo = fopen(argv[3], "wb");
  fwrite(out.data(), 8, out.size(), fo);
  fclose(fo);
  fo = fopen(argv[4], "wb");
  fwrite(nrm.data(), 8, nrm.size(), fo);
  fclose(fo);
  return 0;
}
