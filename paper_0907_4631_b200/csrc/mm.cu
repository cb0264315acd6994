// mm.cu — Matrix Market ingestion (host code): user-supplied sparse matrices (the paper's UF
// collection matrices, are distributed in this format) become the CSR operand of
// phipm_solve_csr / phipm_solve_csr_host.
//
// Supported: "%%MatrixMarket matrix coordinate {real|integer|pattern} {general|symmetric|
// skew-symmetric}", square.  Output: CSR with columns ascending within each row; duplicate
// entries are summed in file order; symmetric / skew-symmetric storage is expanded (the mirror
// of (i, j, v) is (j, i, v) / (j, i, -v), diagonal entries once).  Indices in the file are 1-based.
#include <algorithm>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "phipm.h"

namespace {

struct MMEntry {
    int64_t r, c;
    double v;
    int64_t seq;               // file order (duplicates are summed in this order)
};

int mm_parse(const char *path, int64_t &n, std::vector<MMEntry> &ent)
{
    FILE *f = fopen(path, "r");
    if (!f) return PHIPM_EINVAL;
    char line[4096];
    if (!fgets(line, sizeof line, f)) { fclose(f); return PHIPM_EINVAL; }
    std::string h(line);
    for (auto &ch : h) ch = (char)tolower((unsigned char)ch);
    if (h.rfind("%%matrixmarket", 0) != 0 || h.find("matrix") == std::string::npos ||
        h.find("coordinate") == std::string::npos) {
        fclose(f);
        return PHIPM_EINVAL;
    }
    const bool pattern = h.find("pattern") != std::string::npos;
    const bool complexv = h.find("complex") != std::string::npos;
    const bool skew = h.find("skew-symmetric") != std::string::npos;
    const bool sym = !skew && h.find("symmetric") != std::string::npos;
    const bool herm = h.find("hermitian") != std::string::npos;
    if (complexv || herm) { fclose(f); return PHIPM_EINVAL; }
    // size line (after comments / blank lines)
    long long M = -1, N = -1, L = -1;
    while (fgets(line, sizeof line, f)) {
        if (line[0] == '%') continue;
        bool blank = true;
        for (char *p = line; *p; p++)
            if (!isspace((unsigned char)*p)) { blank = false; break; }
        if (blank) continue;
        if (sscanf(line, "%lld %lld %lld", &M, &N, &L) != 3) { fclose(f); return PHIPM_EINVAL; }
        break;
    }
    if (M <= 0 || M != N || L < 0 || M >= ((long long)1 << 31)) { fclose(f); return PHIPM_EINVAL; }
    n = M;
    ent.clear();
    ent.reserve((size_t)L * ((sym || skew) ? 2 : 1));
    int64_t seq = 0;
    for (long long k = 0; k < L; k++) {
        long long i, j;
        double v = 1.0;
        int got;
        do {
            if (!fgets(line, sizeof line, f)) { fclose(f); return PHIPM_EINVAL; }
        } while (line[0] == '%');
        got = pattern ? sscanf(line, "%lld %lld", &i, &j) : sscanf(line, "%lld %lld %lf", &i, &j, &v);
        if (got != (pattern ? 2 : 3) || i < 1 || j < 1 || i > M || j > N) { fclose(f); return PHIPM_EINVAL; }
        ent.push_back({i - 1, j - 1, v, seq++});
        if ((sym || skew) && i != j) ent.push_back({j - 1, i - 1, skew ? -v : v, seq++});
        if (skew && i == j) { fclose(f); return PHIPM_EINVAL; }   // skew-symmetric: zero diagonal, not stored
    }
    fclose(f);
    std::stable_sort(ent.begin(), ent.end(), [](const MMEntry &a, const MMEntry &b) {
        return a.r != b.r ? a.r < b.r : a.c < b.c;
    });
    // duplicate (r, c) entries are rejected: a 'symmetric' file that stores both
    // triangles would otherwise double its off-diagonal values silently
    for (size_t k = 1; k < ent.size(); k++)
        if (ent[k - 1].r == ent[k].r && ent[k - 1].c == ent[k].c) return PHIPM_EINVAL;
    if (ent.size() >= ((size_t)1 << 31)) return PHIPM_EINVAL;
    return PHIPM_OK;
}

} // namespace

extern "C" int phipm_mm_read(const char *path, int64_t *n, int64_t *nnz, int32_t *row_ptr, int32_t *col, double *val)
{
    if (!path || !n || !nnz) return PHIPM_EINVAL;
    int64_t nn = 0;
    std::vector<MMEntry> ent;
    const int rc = mm_parse(path, nn, ent);
    if (rc) return rc;
    *n = nn;
    *nnz = (int64_t)ent.size();
    if (!row_ptr && !col && !val) return PHIPM_OK;          // size query
    if (!row_ptr || !col || !val) return PHIPM_EINVAL;
    std::fill(row_ptr, row_ptr + nn + 1, 0);
    for (const auto &e : ent) row_ptr[e.r + 1]++;
    for (int64_t r = 0; r < nn; r++) row_ptr[r + 1] += row_ptr[r];
    for (size_t k = 0; k < ent.size(); k++) {
        col[k] = (int32_t)ent[k].c;
        val[k] = ent[k].v;
    }
    return PHIPM_OK;
}
