"""Generate the Stirling-error table delta(k) = ln k! - [(k + 1/2) ln k - k + ln(2 pi)/2]
for k = 1..15 (CUDA probe generator, Loader's saddle-point form of the Poisson pmf).
Prints C hex-float literals (exactly rounded from 40-digit mpmath values).  CUDA-side tool
only; the oracle evaluates the pmf from its plain definition and never uses this table."""
import mpmath

mpmath.mp.dps = 50
for k in range(0, 16):
    if k == 0:
        v = mpmath.mpf(0)
    else:
        v = mpmath.loggamma(k + 1) - ((k + mpmath.mpf(1) / 2) * mpmath.log(k) - k
                                      + mpmath.log(2 * mpmath.pi) / 2)
    print(f"    {float(v).hex()},  /* k = {k:2d}: {mpmath.nstr(v, 20)} */")
