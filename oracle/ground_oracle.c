/*
 * GROUND-REMOVAL ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of the RANSAC plane-fit ground removal
 * that precedes clustering.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.  It shares no code, header or
 * constant with the CUDA path (paper_2208_07678_b200/csrc/fec_ground.cu).
 *
 * Sources: PAPER.md L179-184 (§2.1: "remove the ground surface as a pre-processing"; plane
 * fitting is one of the methods it names) and SPEC.md L296-323 (module `preprocess`,
 * op remove_ground: sample 3 non-collinear points, count inliers within the threshold,
 * keep the best plane whose normal is within max_tilt of +z, refine by least squares,
 * remove the inliers, keep the survivors' relative order; no plane with >= 10% inliers
 * -> cloud unchanged).  The readings that fix the arithmetic (G1-G7):
 *
 *   hypothesis h = (i0, i1, i2), drawn by the caller (G1); invalid unless all three indices
 *   are in [0, n) and distinct.  In double, every operation IEEE round-to-nearest, no FMA:
 *     u = p1 - p0,  v = p2 - p0
 *     m = u x v = (uy*vz - uz*vy, uz*vx - ux*vz, ux*vy - uy*vx)
 *     L = sqrt((mx*mx + my*my) + mz*mz);  invalid if L == 0 or L is not finite
 *     nrm = m / L  (per component);  if nz < 0: nrm = -nrm
 *     off = -(((nx*p0x) + (ny*p0y)) + (nz*p0z))
 *     tilt-valid iff nz >= cos_max_tilt                                          (G2)
 *   plane_h = (float)(nx, ny, nz, off)   (round to nearest)
 *   residual r(p) = fmaf(nz, z, fmaf(ny, y, fmaf(nx, x, off)))   (binary32, each fmaf
 *     rounded once);  inlier iff |r(p)| <= threshold (binary32)                 (G3)
 *   best = the valid h with the most inliers, the lowest h among equals         (G4)
 *   ground iff best exists and count(best) >= min_inliers                        (G5)
 *   removed = the inliers of plane_best; survivors keep their input order       (G6)
 *
 * Compile: gcc -O2 -ffp-contract=off -fno-fast-math (x86-64 SSE2; fmaf is glibc's correctly
 * rounded fused multiply-add).
 */
#include <math.h>
#include <stdint.h>

/* one hypothesis (G2); returns 1 if the three indices give a plane (valid or not for tilt),
 * writes the binary32 plane and the tilt flag */
int oracle_ground_plane(const float* points, int64_t n, const int32_t* tri, double cos_max_tilt,
                        float* plane_out, int32_t* tilt_ok) {
    plane_out[0] = plane_out[1] = plane_out[2] = plane_out[3] = 0.0f;
    *tilt_ok = 0;
    int32_t a = tri[0], b = tri[1], c = tri[2];
    if (a < 0 || b < 0 || c < 0 || a >= n || b >= n || c >= n) return 0;
    if (a == b || a == c || b == c) return 0;
    double p0x = points[3 * (int64_t)a], p0y = points[3 * (int64_t)a + 1], p0z = points[3 * (int64_t)a + 2];
    double p1x = points[3 * (int64_t)b], p1y = points[3 * (int64_t)b + 1], p1z = points[3 * (int64_t)b + 2];
    double p2x = points[3 * (int64_t)c], p2y = points[3 * (int64_t)c + 1], p2z = points[3 * (int64_t)c + 2];
    double ux = p1x - p0x, uy = p1y - p0y, uz = p1z - p0z;
    double vx = p2x - p0x, vy = p2y - p0y, vz = p2z - p0z;
    double t1, t2;
    t1 = uy * vz; t2 = uz * vy; double mx = t1 - t2;
    t1 = uz * vx; t2 = ux * vz; double my = t1 - t2;
    t1 = ux * vy; t2 = uy * vx; double mz = t1 - t2;
    double sx = mx * mx, sy = my * my, sz = mz * mz;
    double s = sx + sy;
    s = s + sz;
    double L = sqrt(s);
    if (!(L > 0.0) || !isfinite(L)) return 0;
    double nx = mx / L, ny = my / L, nz = mz / L;
    if (nz < 0.0) { nx = -nx; ny = -ny; nz = -nz; }
    double q = nx * p0x;
    double r = ny * p0y;
    q = q + r;
    r = nz * p0z;
    q = q + r;
    double off = -q;
    plane_out[0] = (float)nx;
    plane_out[1] = (float)ny;
    plane_out[2] = (float)nz;
    plane_out[3] = (float)off;
    *tilt_ok = nz >= cos_max_tilt;
    return 1;
}

/* G3 */
float oracle_ground_residual(const float* plane, const float* p) {
    float r = fmaf(plane[0], p[0], plane[3]);
    r = fmaf(plane[1], p[1], r);
    r = fmaf(plane[2], p[2], r);
    return r;
}

int oracle_ground_is_inlier(const float* plane, const float* p, float threshold) {
    return fabsf(oracle_ground_residual(plane, p)) <= threshold;
}

/* all hypotheses: planes [H][4], valid[H] (plane exists and tilt ok), counts[H] (inliers of
 * every plane that exists; 0 otherwise) */
void oracle_ground_counts(const float* points, int64_t n, const int32_t* triplets, int32_t H, float threshold,
                          double cos_max_tilt, float* planes, int32_t* valid, int64_t* counts) {
    for (int32_t h = 0; h < H; ++h) {
        int32_t tilt_ok = 0;
        int ok = oracle_ground_plane(points, n, triplets + 3 * (int64_t)h, cos_max_tilt, planes + 4 * (int64_t)h,
                                     &tilt_ok);
        valid[h] = ok && tilt_ok;
        int64_t c = 0;
        if (ok)
            for (int64_t i = 0; i < n; ++i) c += oracle_ground_is_inlier(planes + 4 * (int64_t)h, points + 3 * i, threshold);
        counts[h] = c;
    }
}

/* inlier mask of one plane; returns the count */
int64_t oracle_ground_mask(const float* points, int64_t n, const float* plane, float threshold, uint8_t* mask) {
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i) {
        mask[i] = (uint8_t)oracle_ground_is_inlier(plane, points + 3 * i, threshold);
        c += mask[i];
    }
    return c;
}
