"""Mutation check for the oracle pins: apply plausible mistakes (dropped term, wrong sign,
wrong index, transposed operand, wrong factor order) to oracle/oqr_oracle.c one at a time,
rebuild, and confirm that tests/test_oracle_pins.py fails for each.  Restores the source.

    python tests/oracle_mutation_check.py   (test infrastructure: not collected by pytest)
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oqr_oracle.c")

MUTATIONS = {
    "gram_transposed_A": ("b[i] += acol[i] * z;", "b[i] += A[i * lda + j] * z;"),
    "gram_drop_last_j": ("for (int64_t j = 0; j < m; j++) {\n      const double* acol",
                         "for (int64_t j = 0; j < m - 1; j++) {\n      const double* acol"),
    "potrf_sign": ("double d = G[j * ldg + j] - dot;", "double d = G[j * ldg + j] + dot;"),
    "potrf_index": ("s += R[j * ldr + k] * R[l * ldr + k];", "s += R[j * ldr + k] * R[l * ldr + k + (k+1<j)];"),
    "trsm_index": ("s += q[k] * R[j * ldr + k];", "s += q[k] * R[k * ldr + j];"),
    "trsm_drop_div": ("q[j] = (Z[j * ldz + i] - s) / R[j * ldr + j];", "q[j] = (Z[j * ldz + i] - s);"),
    "trmm_order": ("s += R2[k * ld2 + i] * R1[j * ld1 + k];", "s += R1[k * ld1 + i] * R2[j * ld2 + k];"),
    "prequr_RUS_order": ("else orc_trmm(n, U, n, S, n, R, n);", "else orc_trmm(n, S, n, U, n, R, n);"),
    "normal2_R_order": ("else orc_trmm(n, R2, n, R1, n, R, n);", "else orc_trmm(n, R1, n, R2, n, R, n);"),
    "normal2_Q1_not_used": ("int info2 = orc_normal(m, n, A, lda, Q1, m, Q, R2);",
                            "int info2 = orc_normal(m, n, A, lda, Z, ldz, Q, R2);"),
    "prequr_Y_skipped": ("int info2 = orc_normal(m, n, A, lda, Y, m, Q, U);",
                         "int info2 = orc_normal(m, n, A, lda, Z, ldz, Q, U);"),
    "euclid_gram_index": ("s += zk[i] * zl[i];", "s += zk[i] * zk[i];"),
    # the double-double checkers (tests/test_oracle_checkers.py)
    "dd_drop_product_error": ("double lo = s.lo + acc.lo + pe;", "double lo = s.lo + acc.lo;"),
    "dd_two_sum_drop_b_part": ("dd_t r = {s, (a - (s - bb)) + (b - bb)};", "dd_t r = {s, (a - (s - bb))};"),
    "dd_drop_lo_of_dd_operand": ("double t = a * b.lo;", "double t = 0.0 * b.lo;"),
    "dd_gram_M_no_fabs_A": ("sa += fabs(a) * fabs(z);", "sa += a * fabs(z);"),
    "dd_gram_M_no_fabs_Z": ("sa += fabs(Z[k * ldz + i]) * Babs[l * m + i];", "sa += Z[k * ldz + i] * Babs[l * m + i];"),
    "dd_gram_transposed_A": ("double a = A[j * lda + i], z = Z[l * ldz + j];", "double a = A[i * lda + j], z = Z[l * ldz + j];"),
    "dd_resid_k_range": ("for (int64_t k = 0; k <= j; k++) {\n        double q", "for (int64_t k = 0; k < j; k++) {\n        double q"),
    "dd_resid_sign": ("s = dd_add_prod(s, -q, r);", "s = dd_add_prod(s, q, r);"),
    "dd_resid_QRabs_no_fabs": ("sa += fabs(q) * fabs(r);", "sa += q * fabs(r);"),
    "dd_chol_resid_p_range": ("for (int64_t p = 0; p <= kmax; p++)", "for (int64_t p = 0; p < kmax; p++)"),
    "dd_chol_resid_index": ("double a = R[k * ldr + p], b = R[l * ldr + p];", "double a = R[k * ldr + p], b = R[l * ldr + k];"),
    "dd_orth_missing_minus_I": ("dd_t s = {k == l ? -1.0 : 0.0, 0.0};\n      for (int64_t i = 0; i < m; i++) s = dd_add_dd_prod(s, Q[k * ldq + i], AQ[l * m + i]);\n      E[l * n + k] = s.hi + s.lo;\n    }\n  free(AQ);\n}\n\n/* G = Z",
                                "dd_t s = {0.0, 0.0};\n      for (int64_t i = 0; i < m; i++) s = dd_add_dd_prod(s, Q[k * ldq + i], AQ[l * m + i]);\n      E[l * n + k] = s.hi + s.lo;\n    }\n  free(AQ);\n}\n\n/* G = Z"),
    "dd_orth_transposed_A": ("s = dd_add_prod(s, A[j * lda + i], Q[l * ldq + j]);", "s = dd_add_prod(s, A[i * lda + j], Q[l * ldq + j]);"),
    "dd_orth_cols_wrong_col": ("const double q = Q[cols[l] * ldq + j];", "const double q = Q[l * ldq + j];"),
    # the Householder pre-step (tests/test_oracle_hh.py)
    "hh_beta_sign": ("const double beta = alpha >= 0.0 ? -nrm : nrm;", "const double beta = alpha >= 0.0 ? nrm : -nrm;"),
    "hh_tau": ("tau[j] = (beta - alpha) / beta;", "tau[j] = (beta - alpha) / alpha;"),
    "hh_tail_from_diag": ("for (int64_t i = j + 1; i < m; i++) tail += xj[i] * xj[i];",
                          "for (int64_t i = j + 2; i < m; i++) tail += xj[i] * xj[i];"),
    "hh_update_drop_diag_term": ("double w = xl[j];\n      for", "double w = 0.0;\n      for"),
    "hh_org2r_forward_order": ("for (int64_t j = n - 1; j >= 0; j--) {\n    const double* v = X + j * ldx;",
                               "for (int64_t jj = 0; jj < n; jj++) {\n    const int64_t j = jj;\n    const double* v = X + j * ldx;"),
    "hh_org2r_cols_from_0": ("for (int64_t l = j; l < n; l++) {\n      double* y = Y + l * m;",
                             "for (int64_t l = j + 1; l < n; l++) {\n      double* y = Y + l * m;"),
    "hh_sign_fix_row_only": ("for (int64_t i = 0; i < m; i++) Y[j * m + i] = -Y[j * m + i];", ";"),
    "prequr_hh_RUS_order": ("else orc_trmm(n, U, n, S, n, R, n);\n  }\n  free(S); free(U); free(Y);\n  return info;\n}\n\n/* E = Y^T Y",
                            "else orc_trmm(n, S, n, U, n, R, n);\n  }\n  free(S); free(U); free(Y);\n  return info;\n}\n\n/* E = Y^T Y"),
    "dd_orth_euclid_missing_minus_I": ("dd_t s = {k == l ? -1.0 : 0.0, 0.0};\n      for (int64_t i = 0; i < m; i++) s = dd_add_prod(s, Y[k * ldy + i], Y[l * ldy + i]);",
                                       "dd_t s = {0.0, 0.0};\n      for (int64_t i = 0; i < m; i++) s = dd_add_prod(s, Y[k * ldy + i], Y[l * ldy + i]);"),
    "dd_orth_tridiag_e_index": ("if (i > 0) s = dd_add_prod(s, e[i - 1], q[i - 1]);", "if (i > 0) s = dd_add_prod(s, e[i], q[i - 1]);"),
}


def main():
    orig = open(SRC).read()
    backup = SRC + ".bak"
    shutil.copy(SRC, backup)
    survivors = []
    try:
        for name, (a, b) in MUTATIONS.items():
            assert a in orig, name
            open(SRC, "w").write(orig.replace(a, b, 1))
            r = subprocess.run(
                f'{sys.executable} -c "import oracle; oracle.build(force=True)" && '
                f"{sys.executable} -m pytest tests/test_oracle_pins.py tests/test_oracle_checkers.py "
                f"tests/test_oracle_stable.py tests/test_oracle_tridiag.py tests/test_oracle_hh.py -q -x -p no:cacheprovider 2>&1 | tail -1",
                shell=True, capture_output=True, text=True, cwd=ROOT)
            line = r.stdout.strip()
            killed = "failed" in line
            print(f"{name:24s} {'KILLED ' if killed else 'SURVIVED'}  {line}")
            if not killed:
                survivors.append(name)
    finally:
        shutil.copy(backup, SRC)
        os.remove(backup)
        subprocess.run(f'{sys.executable} -c "import oracle; oracle.build(force=True)"', shell=True, cwd=ROOT)
    print("survivors:", survivors)
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
