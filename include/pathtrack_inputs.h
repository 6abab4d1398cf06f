/* pathtrack_inputs.h -- C-ABI of the host-only inputs library
 * (paper_1501_06625_b200/libpt_inputs.so; no CUDA, never loads the tracker).
 *
 * Everything the hot path consumes or produces as data, each entry citing the
 * reference interface it replaces:
 *
 *   pt_hex_encode_limb / pt_hex_decode_limb / pt_hex_limbs / pt_parse_hex_limbs
 *                           hex_encode_limb, hex_decode_limb, hex_limbs,
 *                           parse_hex_limbs        proj/include/pathtrack/hexio.hpp:16-24,
 *                                                  proj/src/hexio.cpp:21-70
 *   pt_system_parse         parse_system           SPEC.md:147-152 (grammar SPEC.md:197)
 *   pt_system_serialize     serialize_system
 *   pt_solutions_write/read solutions file format  SPEC.md:197 (polysys External Interfaces)
 *   pt_gen_cyclic           cyclic_system          SPEC.md:529-537 (Eq. 5)
 *   pt_gen_augment          augment_with_linear    SPEC.md:547-555 (Eq. 6)
 *   pt_cyclic_degree        cyclic_degree          SPEC.md:538-546 (Table 5)
 *   pt_pieri_*              minor_expand, choose_special_matrix and the
 *                           pattern sequence of pieri_sequence
 *                                                  SPEC.md:583-609 (PAPER.md 4.1, Eqs. 7-8)
 *   pt_gen_gamma            Rng::unit<R>           proj/include/pathtrack/rng.hpp:38-41
 *   pt_gen_unit_complex     unit_complex<R>        proj/include/pathtrack/complex.hpp:141-148
 *
 * Conventions are those of pathtrack_b200.h (limbs, SoA complex vectors,
 * return codes).  Text outputs are malloc'ed NUL-terminated strings released
 * with pt_text_free; systems are pt_sysbuf objects released with
 * pt_sysbuf_free.  Parse errors return PT_E_INVAL and leave "line L, column C:
 * message" in pt_inputs_last_error() (thread-local), the reference's
 * std::invalid_argument text where it has one (hexio.cpp:33,37,57,64,68).
 */
#ifndef PATHTRACK_INPUTS_H
#define PATHTRACK_INPUTS_H

#include <stdint.h>

#include "pathtrack_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pt_sysbuf pt_sysbuf;

const char* pt_inputs_last_error(void);
void pt_text_free(char* text);

/* ---- hex limbs (hexio.hpp) ------------------------------------------------ */
/* 16 lowercase hex digits of the binary64 bit pattern; out has >= 17 bytes. */
int pt_hex_encode_limb(double value, char* out);
/* exactly 16 hex digits (either case) -> the double with that bit pattern */
int pt_hex_decode_limb(const char* text, int32_t len, double* out);
/* "#(h1 h2 ...)" of `count` limbs; *out malloc'ed */
int pt_hex_limbs(const double* limbs, int32_t count, char** out);
/* parse "#(...)" into at most `cap` limbs; *count = limbs parsed */
int pt_parse_hex_limbs(const char* text, int32_t len, double* out, int32_t cap, int32_t* count);

/* ---- system files (grammar SPEC.md:197) ------------------ */
/* Parse a system file in precision `prec` into canonical form: terms sorted
 * lexicographically by support, duplicate supports merged by coefficient
 * addition (in `prec`), zero coefficients dropped. */
int pt_system_parse(const char* text, pt_prec prec, pt_sysbuf** out);
/* Serialize with hex-limb coefficients (bit-exact round trip). */
int pt_system_serialize(const pt_system_desc* s, pt_prec prec, char** out);

/* ---- solution files ------------------------------------------------------- */
/* count records; record r: t[r], point r (complex vector of length n in the
 * SoA layout, points packed with stride 2*L*n), residual[r], update[r]. */
int pt_solutions_write(int32_t n, pt_prec prec, int32_t count, const double* t, const double* points,
                       const double* residual, const double* update, char** out);
/* Two calls: with points == NULL only *count and *n are returned. */
int pt_solutions_read(const char* text, pt_prec prec, int32_t cap, int32_t* count, int32_t* n, double* t,
                      double* points, double* residual, double* update);

/* ---- synthetic systems (BASELINE.json configs) ---------------------------- */
int pt_gen_cyclic(int32_t n, pt_prec prec, pt_sysbuf** out);
int pt_gen_augment(const pt_sysbuf* f, int32_t dim, uint64_t seed, pt_prec prec, pt_sysbuf** out);
int pt_gen_chandra(int32_t n, double c, pt_prec prec, pt_sysbuf** out);
int pt_gen_random_dense(int32_t n, int32_t degree, int32_t n_monomials, uint64_t seed, pt_prec prec,
                        pt_sysbuf** out);
int pt_gen_total_degree(int32_t n, int32_t degree, pt_prec prec, pt_sysbuf** out);
int pt_sysbuf_desc(const pt_sysbuf* s, pt_system_desc* out);
/* Copy a caller-described system into a new buffer (canonical form enforced). */
int pt_sysbuf_from_desc(const pt_system_desc* d, pt_prec prec, pt_sysbuf** out);
/* Concatenate the equations of a and b (same n_vars, same precision). */
int pt_sysbuf_stack(const pt_sysbuf* a, const pt_sysbuf* b, pt_sysbuf** out);
void pt_sysbuf_free(pt_sysbuf* s);
/* Rng(seed).unit<R>() (rng.hpp:38-41): 2L limbs. */
int pt_gen_gamma(uint64_t seed, pt_prec prec, double* out);
/* unit_complex<R>(theta) (complex.hpp:141-148): 2L limbs. */
int pt_gen_unit_complex(double theta, pt_prec prec, double* out);

/* cyclic_degree (Table 5): n = l m^2 with m >= 2 maximal and l squarefree;
 * returns 1 and fills m, l, dim = m-1, degree = m; 0 when none; <0 on error. */
int pt_cyclic_degree(int32_t n, int32_t* m, int32_t* l, int32_t* dim, int32_t* degree);

/* ---- Pieri homotopies ----------------------------------- */
/* Variable-introduction events of the n x p localization pattern (n = m+p):
 * rightmost column first, top to bottom below its pivot (rows j+1..m+j of
 * column j, 1-based, pivot of column j at row j), then one column left.
 * rows[e], cols[e] (0-based) for e < m*p. */
int pt_pieri_events(int32_t m, int32_t p, int32_t* rows, int32_t* cols);
/* Random input planes A^(1..count): each n x m column-major complex in the
 * SoA layout (stride 2*L*n*m per matrix), entries Rng(seed).box<R>() drawn
 * matrix by matrix, column by column. */
int pt_pieri_planes(int32_t m, int32_t p, int32_t count, uint64_t seed, pt_prec prec, double* out);
/* minor_expand: det([A | X_k]) fully expanded (Laplace over the X columns,
 * complementary m x m minors of A in `prec`), as a one-equation system in
 * the k variables of stage k (variable v = event v). */
int pt_pieri_minor(int32_t m, int32_t p, int32_t k, const double* A, pt_prec prec, pt_sysbuf** out);
/* det([A | X_k(x)]) evaluated numerically at x (k complex, SoA) -> 2L limbs. */
int pt_pieri_det(int32_t m, int32_t p, int32_t k, const double* A, const double* x, pt_prec prec,
                 double* out);
/* Stage 1 is linear in its one variable: x = -det(X_1(0)) / (det(X_1(1)) -
 * det(X_1(0))) for A = A^(1), in `prec` (2L limbs). */
int pt_pieri_linear_start(int32_t m, int32_t p, const double* A, pt_prec prec, double* x);
/* choose_special_matrix for stage k (its new variable = event k-1) at the
 * start point x (k complex, new variable = 0): the first S_X (basis-vector
 * columns, then sums of two basis vectors) with det([S_X|X_k(x)]) == 0 and a
 * nonzero derivative in the new variable; S_X written like A. */
int pt_pieri_special(int32_t m, int32_t p, int32_t k, const double* x, pt_prec prec, double* S);

#ifdef __cplusplus
}
#endif

#endif /* PATHTRACK_INPUTS_H */
