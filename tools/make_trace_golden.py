"""Golden JSONL cases for the trace codec: the REFERENCE's load_trace (trace.py:108-167)
run on each text in this container; records or the TraceError text are recorded.

    python tools/make_trace_golden.py     # writes tests/golden/jsonl_cases.json
"""
import json
import math
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refcompat import import_reference  # noqa: E402

R = '"arrival_s":0.5,"blocks":[1,2,3],"in":40,"out":3'
CASES = {
    "valid": '{"id":1,' + R + ',"class":7}\n{"id":2,"arrival_s":1.25,"blocks":[18446744073709551615],"in":1,"out":1}\n',
    "class_null_and_derived": '{"id":1,' + R + ',"class":null}\n{"id":2,' + R + '}\n',
    "bool_ints": '{"id":true,' + R.replace('"in":40', '"in":true') + ',"class":false}\n',
    "minus_zero": '{"id":-0,"arrival_s":-0.0,"blocks":[-0,5],"in":9,"out":2,"class":-0}\n',
    "arrival_int_inf_nan": '{"id":1,"arrival_s":3,"blocks":[1],"in":1,"out":1}\n{"id":2,"arrival_s":NaN,"blocks":[1],"in":1,"out":1}\n'
                           '{"id":3,"arrival_s":1,"blocks":[1],"in":1,"out":1}\n{"id":4,"arrival_s":1e400,"blocks":[1],"in":1,"out":1}\n'
                           '{"id":5,"arrival_s":Infinity,"blocks":[1],"in":1,"out":1}\n',
    "big_arrival_int": '{"id":1,"arrival_s":123456789012345678901234567890,"blocks":[1],"in":1,"out":1}\n',
    "duplicate_keys": '{"id":1,"id":9,"blocks":"x",' + R + ',"blocks":[4,5]}\n',
    "extra_fields": '{"meta":{"a":[1,{"b":"c\\\\\\"\\u00e9\\ud83d\\ude00"}],"t":true,"n":null},"x":-1.5e-3,' + '"id":1,' + R + '}\n',
    "escaped_key": '{"\\u0069d":4,' + R + '}\n',
    "whitespace": '  {"id" : 1 ,\t"arrival_s" :0.5 , "blocks":[ 1 , 2 ] , "in":20,"out":1 }  \n',
    "blank_lines": '\n   \n\t\n\x1f\n\u00a0\u3000\n{"id":1,' + R + '}\n\n',
    "crlf_cr": '{"id":1,' + R + '}\r\n{"id":2,' + R + '}\r{"id":3,' + R + '}',
    "vt_split": '{"id":1,' + R + '}\x0b{"id":2,' + R + '}\u2028{"id":3,' + R + '}\x1c{"id":4,' + R + '}\x85{"id":5,' + R + '}\n',
    "empty_file": '',
    "json_unclosed": '{"id":1,\n',
    "json_trailing_comma_obj": '{"id":1,}\n',
    "json_trailing_comma_arr": '{"id":1,"blocks":[1,]}\n',
    "json_no_colon": '{"id" 1}\n',
    "json_single_quotes": "{'id':1}\n",
    "json_bad_literal": 'nul\n',
    "json_leading_zero": '{"id":01}\n',
    "json_dot": '{"id":1.}\n',
    "json_unterminated_str": '{"id":"abc\n',
    "json_bad_escape": '{"id":"a\\x"}\n',
    "json_bad_u": '{"id":"\\u12G4"}\n',
    "json_control_char": '{"id":"a\tb"}\n',
    "json_extra_data": '{}x\n',
    "json_bom": '\ufeff{"id":1,' + R + '}\n',
    "json_minus": '{"id":-}\n',
    "json_exp": '{"id":1e}\n',
    "json_missing_comma": '{"id":1 "in":2}\n',
    "json_second_line": '{"id":1,' + R + '}\n{"id":2,' + R + '\n',
    "not_object_array": '[1,2]\n',
    "not_object_num": '5\n',
    "not_object_null": 'null\n',
    "missing_id": '{' + R + '}\n',
    "missing_arrival": '{"id":1,"blocks":[1],"in":1,"out":1}\n',
    "missing_blocks": '{"id":1,"arrival_s":0,"in":1,"out":1}\n',
    "missing_in": '{"id":1,"arrival_s":0,"blocks":[1],"out":1}\n',
    "missing_out": '{"id":1,"arrival_s":0,"blocks":[1],"in":1}\n',
    "id_negative": '{"id":-1,' + R + '}\n',
    "id_float": '{"id":1.5,' + R + '}\n',
    "id_string": '{"id":"1",' + R + '}\n',
    "arrival_negative": '{"id":1,"arrival_s":-1,"blocks":[1],"in":1,"out":1}\n',
    "arrival_bool": '{"id":1,"arrival_s":true,"blocks":[1],"in":1,"out":1}\n',
    "arrival_string": '{"id":1,"arrival_s":"0","blocks":[1],"in":1,"out":1}\n',
    "arrival_neg_inf": '{"id":1,"arrival_s":-Infinity,"blocks":[1],"in":1,"out":1}\n',
    "blocks_empty": '{"id":1,"arrival_s":0,"blocks":[],"in":1,"out":1}\n',
    "blocks_string": '{"id":1,"arrival_s":0,"blocks":"x","in":1,"out":1}\n',
    "blocks_float": '{"id":1,"arrival_s":0,"blocks":[1.0],"in":1,"out":1}\n',
    "blocks_negative": '{"id":1,"arrival_s":0,"blocks":[1,-1],"in":1,"out":1}\n',
    "blocks_too_big": '{"id":1,"arrival_s":0,"blocks":[18446744073709551616],"in":1,"out":1}\n',
    "blocks_nested": '{"id":1,"arrival_s":0,"blocks":[[1]],"in":1,"out":1}\n',
    "in_zero": '{"id":1,"arrival_s":0,"blocks":[1],"in":0,"out":1}\n',
    "in_float": '{"id":1,"arrival_s":0,"blocks":[1],"in":1.0,"out":1}\n',
    "out_false": '{"id":1,"arrival_s":0,"blocks":[1],"in":1,"out":false}\n',
    "class_negative": '{"id":1,' + R + ',"class":-1}\n',
    "class_too_big": '{"id":1,' + R + ',"class":18446744073709551616}\n',
    "class_float": '{"id":1,' + R + ',"class":1.5}\n',
    "class_string": '{"id":1,' + R + ',"class":"c"}\n',
    "order_violation": '{"id":1,"arrival_s":2.5,"blocks":[1],"in":1,"out":1}\n\n{"id":2,"arrival_s":0.1,"blocks":[1],"in":1,"out":1}\n',
    "order_equal_ok": '{"id":1,"arrival_s":2.5,"blocks":[1],"in":1,"out":1}\n{"id":2,"arrival_s":2.5,"blocks":[1],"in":1,"out":1}\n',
}


def _f(x):
    return repr(float(x))


def main():
    import_reference()
    from routesim.trace import TraceError, load_trace
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, text in CASES.items():
            p = os.path.join(d, name + ".jsonl")
            with open(p, "w", encoding="utf-8", newline="") as fh:
                fh.write(text)
            try:
                recs = load_trace(p)
                out[name] = {"text": text, "records": [[int(r.request_id), _f(r.arrival_s), [int(b) for b in r.prefix_blocks],
                                                        int(r.input_tokens), int(r.output_tokens), int(r.class_key)]
                                                       for r in recs]}
            except TraceError as exc:
                out[name] = {"text": text, "error": str(exc), "line": exc.line}
            print(name, "error" in out[name] and out[name]["error"] or len(out[name]["records"]))
    with open(os.path.join(ROOT, "tests", "golden", "jsonl_cases.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
