"""Parity comparator for feature tables.

* Bit-exact columns must be identical (==): labels and the 24 intensity columns
  derived from exact integer sums / the sorted multiset.
* Every other column must satisfy  |g - r| <= tol * (max(|g|, |r|) + s)
  with tol = 1e-9 for intensity and moments, 1e-6 for Haralick (north star),
  and s a per-feature natural scale:
    - central moments mu_pq: s = sum w (lx + lcx)^p (ly + lcy)^q, lx = x - bbox.x_min,
      lcx = the local centroid.  This is the magnitude of the terms of the
      reference's own binomial shift from the bbox origin (moments.cpp:69-79),
      i.e. the scale of ITS rounding error: against exact rational truth the
      reference misses a pure relative bound by up to 8.6e-8 (weighted mu33 on a
      Siemens-star ROI, tests/golden/blobs_star) and 2.4e-8.  The
      device path itself is checked against exact rational truth at 1e-12 of the
      natural scale sum w |x-cx|^p |y-cy|^q in test_gpu_parity.py.
    - eta_pq: s_mu / m00^(1+(p+q)/2);  Hu: s2, s2^2, s3^2, s3^2, s3^4, s2*s3^2, s3^4
      with s2 = e20+e02+2e11, s3 = e30+3e12+3e21+e03 over e = |eta| + s_eta
    - skewness / hyperskewness, and Haralick clushade / corr / infomeas1: s = 1
    - Haralick clutend / cluprom: s = d^k / tol, d = c u (|sumave| + 1), the
      rounding noise of mu_x + mu_y raised to the moment's power (their truth is
      0 when every pair sums to the same level); difvar / sumvar likewise with
      difave / sumave;
      clushade: c u sqrt(clutend cluprom) / tol (its terms cancel between signs);
      entropies (entropy, je, sument, difentro): c u (H + 16) / tol (a one-cell
      distribution is exactly 0 from integer counts, ~u from summed p)
    - an _ave column inherits the mean of its angle columns' bounds
    - Haralick infomeas2 = sqrt(1 - exp(-2 (HXY2 - HXY))): a rounding error d of
      order c u (HXY + 1) in the entropy difference moves it by d / imc2 (by
      sqrt(d) near 0), so s = d / (tol max(imc2, sqrt(d))), c = 4096; this only
      matters where HXY2 ~ HXY (e.g. two-level ROIs, imc2 near 0)
    - everything else: s = 1e-300 (pure relative)
"""
from __future__ import annotations

import numpy as np

EXACT_INTENSITY = ["mean", "median", "mode", "min", "max", "range", "median_ad", "iqr", "p1",
                   "p10", "p25", "p75", "p90", "p99", "energy", "rms", "qcod",
                   "integrated_intensity", "edge_mean", "edge_min", "edge_max",
                   "edge_integrated", "weighted_centroid_x", "weighted_centroid_y"]
# shape: everything but orientation (atan2) and the Feret diameters (hypot),
# whose libm implementations differ in the last ulp between CUDA and glibc
EXACT_SHAPE = ["area", "perimeter", "bbox_x", "bbox_y", "bbox_w", "bbox_h", "centroid_x",
               "centroid_y", "circularity", "extent", "aspect_ratio", "convex_area", "solidity",
               "equivalent_diameter", "major_axis_len", "minor_axis_len", "eccentricity",
               "elongation", "euler_number"] + [
               f"extrema_{c}_{a}" for c in ("topleft", "topright", "righttop", "rightbottom",
                                            "bottomright", "bottomleft", "leftbottom", "lefttop")
               for a in ("x", "y")]
EXACT = {"intensity_" + n for n in EXACT_INTENSITY} | {"shape_" + n for n in EXACT_SHAPE}
UNIT_FLOOR = {"intensity_skewness", "intensity_hyperskewness", "shape_orientation"}
HARALICK_UNIT = ("clushade", "corr", "infomeas1")


def _moment_scales(intensity, labels, roi_labels, reference_frame=True):
    """Per ROI, binary and weighted: s_pq = sum w (lx+lcx)^p (ly+lcy)^q (the
    reference's binomial-shift scale) or, with reference_frame=False, the
    natural scale sum w |x-cx|^p |y-cy|^q.  Vectorised over all ROIs (bincount),
    so full-size images (C2: 50k ROIs, 14M pixels) take seconds."""
    roi_labels = np.asarray(roi_labels)
    out = np.zeros((len(roi_labels), 2, 4, 4))
    if len(roi_labels) == 0:
        return out
    ys, xs = np.nonzero(labels)
    lab = labels[ys, xs]
    keep = np.isin(lab, roi_labels)
    ys, xs, lab = ys[keep], xs[keep], lab[keep]
    k = np.searchsorted(roi_labels, lab)
    n = len(roi_labels)
    x, y = xs.astype(np.float64), ys.astype(np.float64)
    val = intensity[ys, xs].astype(np.float64)
    xmin = np.full(n, np.inf)
    ymin = np.full(n, np.inf)
    np.minimum.at(xmin, k, x)
    np.minimum.at(ymin, k, y)
    for g, w in enumerate((np.ones_like(val), val)):
        m = np.bincount(k, w, minlength=n)
        with np.errstate(divide="ignore", invalid="ignore"):
            if reference_frame:
                lx, ly = x - xmin[k], y - ymin[k]
                ax = lx + (np.bincount(k, w * lx, minlength=n) / m)[k]
                ay = ly + (np.bincount(k, w * ly, minlength=n) / m)[k]
            else:
                ax = np.abs(x - (np.bincount(k, w * x, minlength=n) / m)[k])
                ay = np.abs(y - (np.bincount(k, w * y, minlength=n) / m)[k])
        ok = (m > 0)[k]
        ax, ay, ww = ax[ok], ay[ok], w[ok]
        kk = k[ok]
        px = [np.ones_like(ax), ax, ax * ax, ax * ax * ax]
        py = [np.ones_like(ay), ay, ay * ay, ay * ay * ay]
        for p in range(4):
            wp = ww * px[p]
            for q in range(4):
                out[:, g, p, q] = np.bincount(kk, wp * py[q], minlength=n)
    return out


def floors(columns, ref_table, intensity=None, labels=None, roi_labels=None):
    """Per-cell floor s (same shape as the table)."""
    s = np.full(ref_table.shape, 1e-300)
    # names repeat when an angle is listed twice: walk every index, look partners
    # up by name (a repeated angle's columns hold identical values)
    col = {c: i for i, c in enumerate(columns)}
    for i, c in enumerate(columns):
        if c in UNIT_FLOOR:
            s[:, i] = 1.0
        if c.startswith("glcm_") and any(c.startswith("glcm_" + h + "_") for h in HARALICK_UNIT):
            s[:, i] = 1.0
    for i, c in enumerate(columns):
        if c.startswith("glcm_infomeas2_"):
            h = col.get("glcm_entropy_" + c[len("glcm_infomeas2_"):])
            if h is None:
                continue
            d = 4096 * 2.2e-16 * (np.abs(ref_table[:, h]) + 1.0)
            s[:, i] = d / (1e-6 * np.maximum(np.abs(ref_table[:, i]), np.sqrt(d)))
        # entropies -sum p log2 p: when the reference's p sum to 1 only within rounding,
        # a one-cell distribution gives ~u instead of 0 (and the device's integer p give
        # exactly 0); noise c u (H + 16)
        if any(c.startswith(f"glcm_{e}_") for e in ("difentro", "sument", "entropy", "je")):
            s[:, i] = np.maximum(s[:, i], 4096 * 2.2e-16 * (np.abs(ref_table[:, i]) + 16.0) / 1e-6)
        # difvar = sum p (d - difave)^2, sumvar = sum p (k - sumave)^2: rounding noise
        # of the mean, squared (as clutend)
        for v_, m_ in (("difvar", "difave"), ("sumvar", "sumave")):
            if c.startswith(f"glcm_{v_}_"):
                h = col.get(f"glcm_{m_}_" + c[len(f"glcm_{v_}_"):])
                if h is not None:
                    d = 4096 * 2.2e-16 * (np.abs(ref_table[:, h]) + 1.0)
                    s[:, i] = np.maximum(s[:, i], d * d / 1e-6)
        # clushade = sum p s^3 cancels between signs: the noise is u times the terms'
        # magnitude, sum p |s|^3 <= sqrt(clutend cluprom) (Cauchy-Schwarz)
        if c.startswith("glcm_clushade_"):
            sfx = c[len("glcm_clushade_"):]
            ht, hp = col.get("glcm_clutend_" + sfx), col.get("glcm_cluprom_" + sfx)
            if ht is not None and hp is not None:
                mag = np.sqrt(np.abs(ref_table[:, ht]) * np.abs(ref_table[:, hp]))
                s[:, i] = np.maximum(s[:, i], 4096 * 2.2e-16 * mag / 1e-6)
        for k, name in ((2, "clutend"), (4, "cluprom")):
            # sum p (i + j - mu_x - mu_y)^k: when all mass sits on one anti-diagonal
            # the truth is 0 and both sides return the rounding noise of mu_x + mu_y
            # (d, as for infomeas2) to the k-th power; either may be exactly 0
            if c.startswith(f"glcm_{name}_"):
                h = col.get("glcm_sumave_" + c[len(f"glcm_{name}_"):])
                if h is None:
                    continue
                d = 4096 * 2.2e-16 * (np.abs(ref_table[:, h]) + 1.0)
                s[:, i] = np.maximum(s[:, i], d ** k / 1e-6)
    # an _ave column is the mean of its angle columns: it inherits their noise, so its
    # bound covers the mean of theirs (e.g. infomeas2 with one angle at ~0, where the
    # noise is sqrt(d), averaged into a larger _ave)
    for i, c in enumerate(columns):
        if not c.endswith("_ave"):
            continue
        pre = c[:-len("ave")]
        j = i - 1
        while j >= 0 and columns[j].startswith(pre) and columns[j][len(pre):].isdigit():
            j -= 1
        ang = list(range(j + 1, i))
        if ang:
            inherited = np.mean([np.abs(ref_table[:, a]) + s[:, a] for a in ang], axis=0) - np.abs(ref_table[:, i])
            s[:, i] = np.maximum(s[:, i], inherited)
    # GLRLM/GLSZM variances sum p (x - mu)^2: the reference's rounding noise scales
    # with E[x^2] (its own lre / hglre / lae / hglze columns), not with the variance.
    # Scale columns are found by position (feature-major blocks, names may repeat
    # when an angle is listed twice).
    feats = ["sre", "lre", "glnu", "glnun", "rlnu", "rlnun", "rp", "glv", "rv", "re", "lglre",
             "hglre", "srlgle", "srhgle", "lrlgle", "lrhgle"]
    for pre, pairs in (("glrlm_", (("glv", "hglre"), ("rv", "lre"))),
                       ("glszm_", (("glv", "hglze"), ("zv", "lae")))):
        idx = [i for i, c in enumerate(columns) if c.startswith(pre)]
        if not idx:
            continue
        per = len(idx) // 16  # angles + 1 (glrlm), 1 (glszm)
        names = feats
        if pre == "glszm_":
            names = ["sae", "lae", "glnu", "glnun", "sznu", "sznun", "zp", "glv", "zv", "ze",
                     "lglze", "hglze", "salgle", "sahgle", "lalgle", "lahgle"]
        for var, scale in pairs:
            dv, ds = names.index(var), names.index(scale)
            for k in range(per):
                i, j = idx[dv * per + k], idx[ds * per + k]
                s[:, i] = np.maximum(s[:, i], np.abs(ref_table[:, j]))
    if "moments_mu00" in col and intensity is not None:
        ms = _moment_scales(intensity, labels, roi_labels)
        for g, pre in enumerate(("", "w")):
            m00 = ref_table[:, col[f"moments_{pre}m00"]]
            with np.errstate(divide="ignore", invalid="ignore"):
                for p in range(4):
                    for q in range(4):
                        s[:, col[f"moments_{pre}mu{p}{q}"]] = np.maximum(ms[:, g, p, q], 1e-300)
                        if p + q >= 2:
                            se = ms[:, g, p, q] / np.power(m00, 1.0 + (p + q) / 2.0)
                            s[:, col[f"moments_{pre}eta{p}{q}"]] = np.where(np.isfinite(se), se, 1.0)
                e = {f"{p}{q}": np.abs(ref_table[:, col[f"moments_{pre}eta{p}{q}"]])
                     + s[:, col[f"moments_{pre}eta{p}{q}"]]
                     for p in range(4) for q in range(4) if p + q >= 2}
                s2 = e["20"] + e["02"] + 2 * e["11"]
                s3 = e["30"] + 3 * e["12"] + 3 * e["21"] + e["03"]
                hs = [s2, s2 ** 2, s3 ** 2, s3 ** 2, s3 ** 4, s2 * s3 ** 2, s3 ** 4]
                for k in range(7):
                    s[:, col[f"moments_{pre}hu{k + 1}"]] = np.maximum(hs[k], 1e-300)
    return s


def compare(columns, gpu, ref, s, tol_int=1e-9, tol_glcm=1e-6):
    """Returns a list of (column, worst ratio, n_bad) for violating columns."""
    bad = []
    g, r = np.asarray(gpu), np.asarray(ref)
    for i, c in enumerate(columns):
        a, b = g[:, i], r[:, i]
        if c in EXACT:
            nb = int(np.count_nonzero(~((a == b) | (np.isnan(a) & np.isnan(b)))))
            if nb:
                bad.append((c, float("inf"), nb))
            continue
        tol = tol_glcm if c.startswith("glcm_") else tol_int
        bound = tol * (np.maximum(np.abs(a), np.abs(b)) + s[:, i])
        err = np.abs(a - b)
        ok = (err <= bound) | (a == b)
        if not ok.all():
            ratio = float(np.max(np.where(ok, 0, err / np.maximum(bound, 1e-300))))
            bad.append((c, ratio, int((~ok).sum())))
    return bad


def assert_parity(columns, gpu_labels, gpu, ref_labels, ref, intensity=None, labels=None):
    assert np.array_equal(np.asarray(gpu_labels), np.asarray(ref_labels)), "label list differs"
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    s = floors(columns, ref, intensity, labels, np.asarray(ref_labels))
    bad = compare(columns, gpu, ref, s)
    assert not bad, "parity violations: " + "; ".join(f"{c} (x{r:.3g}, {n} rows)" for c, r, n in bad[:12])
