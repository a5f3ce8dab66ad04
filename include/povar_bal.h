/* povar_bal.h -- native BAL input path of libpovar.so (C ABI).
 *
 * Replaces the reference's Python token loop and pruning
 * (pkg/src/stratba/bal_io.py):
 *   pv_bal_header / pv_bal_parse  -> parse_bal             bal_io.py:155-203
 *   pv_bal_prune_masks            -> prune_underobserved   bal_io.py:244-278 (the O(n_obs)
 *                                    distinct-camera count; the host applies the masks)
 * Decompression (gzip / bzip2 sniffing, load_bal bal_io.py:229-241) stays in the
 * host language; these functions take the decompressed text.
 *
 * Grammar and errors follow parse_bal exactly: whitespace-separated tokens,
 * universal newlines for line numbers, Python int()/float() token syntax, and the
 * same messages (returned with the 1-based line number of the offending token).
 */
#ifndef POVAR_BAL_H
#define POVAR_BAL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PV_BAL_OK 0
#define PV_BAL_EPARSE 6 /* BalParseError(line, message) */

/* The three header counts.  On PV_BAL_EPARSE, *err_line and err_msg (NUL-
 * terminated, truncated to err_cap) describe the error. */
int pv_bal_header(const char* text, size_t len, int64_t* n_cameras, int64_t* n_points,
                  int64_t* n_observations, int64_t* err_line, char* err_msg, size_t err_cap);

/* Full parse into caller-allocated arrays sized from pv_bal_header:
 * cam_idx, pt_idx (n_obs), meas (n_obs x 2), cams (n_cam x 9), pts (n_pt x 3).
 * n_threads <= 0 uses all hardware threads. */
int pv_bal_parse(const char* text, size_t len, int n_threads, int64_t* cam_idx, int64_t* pt_idx,
                 double* meas, double* cams, double* pts, int64_t* err_line, char* err_msg,
                 size_t err_cap);

/* keep_lm[j] = landmark j is seen by >= min_cameras DISTINCT cameras;
 * cam_seen[i] = camera i observes a kept landmark.  Returns the kept
 * observation count in *n_obs_kept. */
int pv_bal_prune_masks(int64_t n_cameras, int64_t n_points, int64_t n_observations,
                       const int64_t* cam_idx, const int64_t* pt_idx, int64_t min_cameras,
                       uint8_t* keep_lm, uint8_t* cam_seen, int64_t* n_obs_kept);

#ifdef __cplusplus
}
#endif

#endif /* POVAR_BAL_H */
