"""IR of the fused-kernel probes (tools/ew_probe.py, tools/ew_cubin.py)."""

SRC = """
func @affsig(%a: f64, %x: f64, %b: f64) -> f64 {
^entry:
  %m = mul %a, %x
  %s = add %m, %b
  %y = sigmoid %s
  ret %y
}
func @aff(%a: f64, %x: f64, %b: f64) -> f64 {
^entry:
  %m = mul %a, %x
  %s = add %m, %b
  ret %s
}
func @ident(%a: f64, %x: f64, %b: f64) -> f64 {
^entry:
  ret %x
}
"""
