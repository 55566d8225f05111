"""Scalar IR functions shared by the golden generator and the parity tests.

Written in the reference's ``.ssair`` text format; covers every scalar op
the fused kernels lower (forward_ad.py:72-143): arithmetic, transcendentals,
branches, loops with i64 counters, calls, select, relu, pow_int, and the
domain-error sites (div, log).
"""

FUSED_SRC = """
func @two(%a: f64, %b: f64) -> f64 {
^entry:
  %s = add %a, %b
  %t = tanh %s
  ret %t
}

func @sgau(%a: f64, %c: f64) -> f64 {
^entry:
  %p = mul %a, %c
  %y = sigmoid %p
  ret %y
}

func @poly(%x: f64) -> f64 {
^entry:
  %x2 = mul %x, %x
  %x3 = mul %x2, %x
  %t = tanh %x3
  ret %t
}

func @branchy(%x: f64) -> f64 {
^entry:
  %z = const f64 0.0
  %pos = gt %x, %z
  br %pos, ^a(), ^b()
^a:
  %one = const f64 1.0
  %u = add %x, %one
  %l = log %u
  jmp ^join(%l)
^b:
  %n = neg %x
  %e = exp %n
  jmp ^join(%e)
^join(%v: f64):
  ret %v
}

func @gauss(%a: f64, %c: f64) -> f64 {
^entry:
  %p = mul %a, %c
  %n = neg %p
  %e = exp %n
  %one = const f64 1.0
  %d = add %one, %e
  %r = div %one, %d
  ret %r
}

func @affsig(%a: f64, %x: f64, %b: f64) -> f64 {
^entry:
  %m = mul %a, %x
  %s = add %m, %b
  %y = sigmoid %s
  ret %y
}

func @cubeloop(%x: f64) -> f64 {
^entry:
  %i0 = const i64 0
  %n = const i64 3
  %a0 = const f64 1.0
  jmp ^head(%i0, %a0)
^head(%i: i64, %acc: f64):
  %more = lt %i, %n
  br %more, ^body(), ^exit(%acc)
^body:
  %a2 = mul %acc, %x
  %one = const i64 1
  %i2 = add %i, %one
  jmp ^head(%i2, %a2)
^exit(%r: f64):
  ret %r
}

func @powloop3(%x: f64) -> f64 {
^entry:
  %p = pow_int %x {n = 3}
  %q = pow_int %x {n = 0}
  %s = add %p, %q
  ret %s
}

func @relusq(%x: f64) -> f64 {
^entry:
  %r = relu %x
  %s = mul %r, %r
  %h = const f64 0.5
  %t = mul %s, %h
  ret %t
}

func @pick(%a: f64, %b: f64) -> f64 {
^entry:
  %c = lt %a, %b
  %m = select %c, %a, %b
  %e = exp %m
  ret %e
}

func @sq(%t: f64) -> f64 {
^entry:
  %s = mul %t, %t
  ret %s
}

func @callin(%x: f64) -> f64 {
^entry:
  %a = call %x {fn = @sq}
  %b = call %a {fn = @sq}
  ret %b
}

func @divy(%a: f64, %b: f64) -> f64 {
^entry:
  %q = div %a, %b
  ret %q
}

func @mixed(%x: f64, %w: f64, %s: f64) -> f64 {
^entry:
  %p = mul %x, %w
  %q = add %p, %s
  %t = tanh %q
  %u = mul %t, %x
  ret %u
}

func @logp(%x: f64) -> f64 {
^entry:
  %l = log %x
  %s = mul %l, %x
  ret %s
}

func @mapped(%x: tensor<4xf64>, %b: f64) -> f64 {
^entry:
  %y = fused_map %x, %b {fn = @gauss}
  %s = reduce_sum %y {axis = all}
  ret %s
}
"""
