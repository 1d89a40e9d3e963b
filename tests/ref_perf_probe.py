"""TEST INFRASTRUCTURE: evaluate the reference's csv_row / emit_csv /
power_law_fit / best_config (oracle/_ref/libsweep1d_ref.so) in a process
that never imports numpy (loading numpy first makes the reference's
ostringstream path crash in-process). JSON in on stdin,
JSON out on stdout."""
import ctypes as C
import json
import os
import sys

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "libsweep1d_ref.so")


class RefRecord(C.Structure):
    _fields_ = [("equation", C.c_int), ("method", C.c_int), ("scheme", C.c_int), ("mode", C.c_int),
                ("grid_size", C.c_ulonglong), ("block_width", C.c_ulonglong), ("work_factor", C.c_int),
                ("ranks", C.c_int), ("steps", C.c_longlong), ("avg_us_per_step", C.c_double),
                ("setup_us", C.c_double), ("messages_sent", C.c_ulonglong), ("bytes_sent", C.c_ulonglong),
                ("exchange_rounds", C.c_ulonglong), ("virtual_comm_us", C.c_double)]


def main():
    req = json.load(sys.stdin)
    lib = C.CDLL(REF)
    lib.ref_csv_row.argtypes = [C.POINTER(RefRecord), C.c_char_p, C.c_size_t]
    lib.ref_emit_csv.argtypes = [C.POINTER(RefRecord), C.c_size_t, C.c_char_p, C.c_char_p, C.c_size_t]
    dp = C.POINTER(C.c_double)
    lib.ref_power_law_fit.argtypes = [dp, dp, C.c_size_t, dp, dp, dp, C.c_char_p, C.c_size_t]
    lib.ref_best_config.restype = C.c_long
    lib.ref_best_config.argtypes = [C.POINTER(RefRecord), C.c_size_t]
    recs = [RefRecord(*r) for r in req.get("records", [])]
    out = {"rows": []}
    for r in recs:
        buf = C.create_string_buffer(1024)
        lib.ref_csv_row(C.byref(r), buf, 1024)
        out["rows"].append(buf.value.decode())
    if recs:
        arr = (RefRecord * len(recs))(*recs)
        if "emit_path" in req:
            out["emit_status"] = lib.ref_emit_csv(arr, len(recs), req["emit_path"].encode(), None, 0)
        out["best"] = lib.ref_best_config(arr, len(recs))
    fits = []
    for xs, ys in req.get("fits", []):
        n = len(xs)
        X, Y = (C.c_double * n)(*xs), (C.c_double * n)(*ys)
        A, b, r2 = C.c_double(), C.c_double(), C.c_double()
        st = lib.ref_power_law_fit(X, Y, n, C.byref(A), C.byref(b), C.byref(r2), None, 0)
        fits.append([st, A.value, b.value, r2.value])
    out["fits"] = fits
    json.dump(out, sys.stdout)


if __name__ == "__main__":
    main()
