/* generated kernel source; compile with: cc -O3 -ffp-contract=off */
#include <math.h>

/* level 0, 998250 instance(s), 78 result(s) each */
static void nh_elem(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 249562; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[0 + i]];
            const double x1 = x[p[0 + i] + 1];
            const double x2 = x[p[0 + i] + 2];
            const double x3 = x[p[998250 + i]];
            const double x4 = x[p[1996500 + i]];
            const double x5 = x[p[2994750 + i]];
            const double x6 = x[p[3993000 + i]];
            const double x7 = x[p[4991250 + i]];
            const double x8 = x[p[5989500 + i]];
            const double x9 = x[p[0 + i] + 9579];
            const double x10 = x[p[0 + i] + 9580];
            const double x11 = x[p[0 + i] + 9581];
            const double x12 = x[p[6987750 + i]];
            const double x13 = x[p[7986000 + i]];
            const double x14 = x[p[8984250 + i]];
            const double x15 = x[p[9982500 + i]];
            const double x16 = x[p[10980750 + i]];
            const double x17 = x[p[11979000 + i]];
            const double x18 = x[p[12977250 + i]];
            const double x19 = x[p[13975500 + i]];
            const double x20 = x[p[14973750 + i]];
            const double x21 = x[p[15972000 + i]];
            const double t0 = x3 - x0;
            const double t1 = x6 - x0;
            const double t2 = x9 - x0;
            const double t3 = x4 - x1;
            const double t4 = x7 - x1;
            const double t5 = x10 - x1;
            const double t6 = x5 - x2;
            const double t7 = x8 - x2;
            const double t8 = x11 - x2;
            const double t9 = x12*t0 + x15*t1 + x18*t2;
            const double t10 = x13*t0 + x16*t1 + x19*t2;
            const double t11 = x14*t0 + x17*t1 + x20*t2;
            const double t12 = x12*t3 + x15*t4 + x18*t5;
            const double t13 = x13*t3 + x16*t4 + x19*t5;
            const double t14 = x14*t3 + x17*t4 + x20*t5;
            const double t15 = x12*t6 + x15*t7 + x18*t8;
            const double t16 = x13*t6 + x16*t7 + x19*t8;
            const double t17 = x14*t6 + x17*t7 + x20*t8;
            const double t18 = t13*t17 - t14*t16;
            const double t19 = t14*t15 - t12*t17;
            const double t20 = t12*t16 - t13*t15;
            const double t21 = t18*t9 + t19*t10 + t20*t11;
            const double t22 = t18/t21;
            const double t23 = (t11*t16 - t10*t17)/t21;
            const double t24 = (t10*t14 - t11*t13)/t21;
            const double t25 = t19/t21;
            const double t26 = (t9*t17 - t11*t15)/t21;
            const double t27 = (t11*t12 - t9*t14)/t21;
            const double t28 = t20/t21;
            const double t29 = (t10*t15 - t9*t16)/t21;
            const double t30 = (t9*t13 - t10*t12)/t21;
            const double t31 = 1.0 - log(t21)*10.0;
            const double t32 = t22*t31;
            const double t33 = t22*10.0;
            const double t34 = t32*t22 + t33*t22 + 1.0;
            const double t35 = t32*t25 + t33*t25;
            const double t36 = t32*t28 + t33*t28;
            const double t37 = t23*t31;
            const double t38 = t37*t22 + t33*t23;
            const double t39 = t37*t25 + t33*t26;
            const double t40 = t37*t28 + t33*t29;
            const double t41 = t24*t31;
            const double t42 = t41*t22 + t33*t24;
            const double t43 = t41*t25 + t33*t27;
            const double t44 = t41*t28 + t33*t30;
            const double t45 = t25*t31;
            const double t46 = t25*10.0;
            const double t47 = t45*t22 + t46*t22;
            const double t48 = t45*t25 + t46*t25 + 1.0;
            const double t49 = t45*t28 + t46*t28;
            const double t50 = t26*t31;
            const double t51 = t50*t22 + t46*t23;
            const double t52 = t50*t25 + t46*t26;
            const double t53 = t50*t28 + t46*t29;
            const double t54 = t27*t31;
            const double t55 = t54*t22 + t46*t24;
            const double t56 = t54*t25 + t46*t27;
            const double t57 = t54*t28 + t46*t30;
            const double t58 = t28*t31;
            const double t59 = t28*10.0;
            const double t60 = t58*t22 + t59*t22;
            const double t61 = t58*t25 + t59*t25;
            const double t62 = t58*t28 + t59*t28 + 1.0;
            const double t63 = t29*t31;
            const double t64 = t63*t22 + t59*t23;
            const double t65 = t63*t25 + t59*t26;
            const double t66 = t63*t28 + t59*t29;
            const double t67 = t30*t31;
            const double t68 = t67*t22 + t59*t24;
            const double t69 = t67*t25 + t59*t27;
            const double t70 = t67*t28 + t59*t30;
            const double t71 = t23*10.0;
            const double t72 = t32*t23 + t71*t22;
            const double t73 = t32*t26 + t71*t25;
            const double t74 = t32*t29 + t71*t28;
            const double t75 = t37*t23 + t71*t23 + 1.0;
            const double t76 = t37*t26 + t71*t26;
            const double t77 = t37*t29 + t71*t29;
            const double t78 = t41*t23 + t71*t24;
            const double t79 = t41*t26 + t71*t27;
            const double t80 = t41*t29 + t71*t30;
            const double t81 = t26*10.0;
            const double t82 = t45*t23 + t81*t22;
            const double t83 = t45*t26 + t81*t25;
            const double t84 = t45*t29 + t81*t28;
            const double t85 = t50*t23 + t81*t23;
            const double t86 = t50*t26 + t81*t26 + 1.0;
            const double t87 = t50*t29 + t81*t29;
            const double t88 = t54*t23 + t81*t24;
            const double t89 = t54*t26 + t81*t27;
            const double t90 = t54*t29 + t81*t30;
            const double t91 = t29*10.0;
            const double t92 = t58*t23 + t91*t22;
            const double t93 = t58*t26 + t91*t25;
            const double t94 = t58*t29 + t91*t28;
            const double t95 = t63*t23 + t91*t23;
            const double t96 = t63*t26 + t91*t26;
            const double t97 = t63*t29 + t91*t29 + 1.0;
            const double t98 = t67*t23 + t91*t24;
            const double t99 = t67*t26 + t91*t27;
            const double t100 = t67*t29 + t91*t30;
            const double t101 = t24*10.0;
            const double t102 = t32*t24 + t101*t22;
            const double t103 = t32*t27 + t101*t25;
            const double t104 = t32*t30 + t101*t28;
            const double t105 = t37*t24 + t101*t23;
            const double t106 = t37*t27 + t101*t26;
            const double t107 = t37*t30 + t101*t29;
            const double t108 = t41*t24 + t101*t24 + 1.0;
            const double t109 = t41*t27 + t101*t27;
            const double t110 = t41*t30 + t101*t30;
            const double t111 = t27*10.0;
            const double t112 = t45*t24 + t111*t22;
            const double t113 = t45*t27 + t111*t25;
            const double t114 = t45*t30 + t111*t28;
            const double t115 = t50*t24 + t111*t23;
            const double t116 = t50*t27 + t111*t26;
            const double t117 = t50*t30 + t111*t29;
            const double t118 = t54*t24 + t111*t24;
            const double t119 = t54*t27 + t111*t27 + 1.0;
            const double t120 = t54*t30 + t111*t30;
            const double t121 = t30*10.0;
            const double t122 = t58*t24 + t121*t22;
            const double t123 = t58*t27 + t121*t25;
            const double t124 = t58*t30 + t121*t28;
            const double t125 = t63*t24 + t121*t23;
            const double t126 = t63*t27 + t121*t26;
            const double t127 = t63*t30 + t121*t29;
            const double t128 = t67*t24 + t121*t24;
            const double t129 = t67*t27 + t121*t27;
            const double t130 = t67*t30 + t121*t30 + 1.0;
            const double t131 = -(x18 + (x12 + x15));
            const double t132 = -(x19 + (x13 + x16));
            const double t133 = -(x20 + (x14 + x17));
            const double t134 = x13*t35 + x12*t34 + x14*t36;
            const double t135 = x16*t35 + x15*t34 + x17*t36;
            const double t136 = x19*t35 + x18*t34 + x20*t36;
            const double t137 = x12*t47 + x13*t48 + x14*t49;
            const double t138 = x15*t47 + x16*t48 + x17*t49;
            const double t139 = x18*t47 + x19*t48 + x20*t49;
            const double t140 = x12*t60 + x13*t61 + x14*t62;
            const double t141 = x15*t60 + x16*t61 + x17*t62;
            const double t142 = x18*t60 + x19*t61 + x20*t62;
            const double t143 = x12*t38 + x13*t39 + x14*t40;
            const double t144 = x15*t38 + x16*t39 + x17*t40;
            const double t145 = x18*t38 + x19*t39 + x20*t40;
            const double t146 = x12*t51 + x13*t52 + x14*t53;
            const double t147 = x15*t51 + x16*t52 + x17*t53;
            const double t148 = x18*t51 + x19*t52 + x20*t53;
            const double t149 = x12*t64 + x13*t65 + x14*t66;
            const double t150 = x15*t64 + x16*t65 + x17*t66;
            const double t151 = x18*t64 + x19*t65 + x20*t66;
            const double t152 = x12*t42 + x13*t43 + x14*t44;
            const double t153 = x15*t42 + x16*t43 + x17*t44;
            const double t154 = x18*t42 + x19*t43 + x20*t44;
            const double t155 = x12*t55 + x13*t56 + x14*t57;
            const double t156 = x15*t55 + x16*t56 + x17*t57;
            const double t157 = x18*t55 + x19*t56 + x20*t57;
            const double t158 = x12*t68 + x13*t69 + x14*t70;
            const double t159 = x15*t68 + x16*t69 + x17*t70;
            const double t160 = x18*t68 + x19*t69 + x20*t70;
            const double t161 = x15*t72 + x16*t73 + x17*t74;
            const double t162 = x18*t72 + x19*t73 + x20*t74;
            const double t163 = x15*t82 + x16*t83 + x17*t84;
            const double t164 = x18*t82 + x19*t83 + x20*t84;
            const double t165 = x15*t92 + x16*t93 + x17*t94;
            const double t166 = x18*t92 + x19*t93 + x20*t94;
            const double t167 = x13*t76 + x12*t75 + x14*t77;
            const double t168 = x16*t76 + x15*t75 + x17*t77;
            const double t169 = x19*t76 + x18*t75 + x20*t77;
            const double t170 = x12*t85 + x13*t86 + x14*t87;
            const double t171 = x15*t85 + x16*t86 + x17*t87;
            const double t172 = x18*t85 + x19*t86 + x20*t87;
            const double t173 = x12*t95 + x13*t96 + x14*t97;
            const double t174 = x15*t95 + x16*t96 + x17*t97;
            const double t175 = x18*t95 + x19*t96 + x20*t97;
            const double t176 = x12*t78 + x13*t79 + x14*t80;
            const double t177 = x15*t78 + x16*t79 + x17*t80;
            const double t178 = x18*t78 + x19*t79 + x20*t80;
            const double t179 = x12*t88 + x13*t89 + x14*t90;
            const double t180 = x15*t88 + x16*t89 + x17*t90;
            const double t181 = x18*t88 + x19*t89 + x20*t90;
            const double t182 = x12*t98 + x13*t99 + x14*t100;
            const double t183 = x15*t98 + x16*t99 + x17*t100;
            const double t184 = x18*t98 + x19*t99 + x20*t100;
            const double t185 = x15*t102 + x16*t103 + x17*t104;
            const double t186 = x18*t102 + x19*t103 + x20*t104;
            const double t187 = x15*t112 + x16*t113 + x17*t114;
            const double t188 = x18*t112 + x19*t113 + x20*t114;
            const double t189 = x15*t122 + x16*t123 + x17*t124;
            const double t190 = x18*t122 + x19*t123 + x20*t124;
            const double t191 = x15*t105 + x16*t106 + x17*t107;
            const double t192 = x18*t105 + x19*t106 + x20*t107;
            const double t193 = x15*t115 + x16*t116 + x17*t117;
            const double t194 = x18*t115 + x19*t116 + x20*t117;
            const double t195 = x15*t125 + x16*t126 + x17*t127;
            const double t196 = x18*t125 + x19*t126 + x20*t127;
            const double t197 = x13*t109 + x12*t108 + x14*t110;
            const double t198 = x16*t109 + x15*t108 + x17*t110;
            const double t199 = x19*t109 + x18*t108 + x20*t110;
            const double t200 = x12*t118 + x13*t119 + x14*t120;
            const double t201 = x15*t118 + x16*t119 + x17*t120;
            const double t202 = x18*t118 + x19*t119 + x20*t120;
            const double t203 = x12*t128 + x13*t129 + x14*t130;
            const double t204 = x15*t128 + x16*t129 + x17*t130;
            const double t205 = x18*t128 + x19*t129 + x20*t130;
            x[10509348 + i] = x21*((t131*t60 + t132*t61 + t133*t62)*t133 + ((t131*t34 + t132*t35 + t133*t36)*t131 + (t132*t48 + t131*t47 + t133*t49)*t132));
            x[11507598 + i] = x21*(t133*(t131*t64 + t132*t65 + t133*t66) + (t131*(t131*t38 + t132*t39 + t133*t40) + t132*(t131*t51 + t132*t52 + t133*t53)));
            x[12505848 + i] = x21*(t133*(t131*t68 + t132*t69 + t133*t70) + (t131*(t131*t42 + t132*t43 + t133*t44) + t132*(t131*t55 + t132*t56 + t133*t57)));
            x[13504098 + i] = (t131*t134 + t132*t137 + t140*t133)*x21;
            x[14502348 + i] = (t143*t131 + t146*t132 + t149*t133)*x21;
            x[15500598 + i] = (t152*t131 + t155*t132 + t158*t133)*x21;
            x[16498848 + i] = (t131*t135 + t132*t138 + t141*t133)*x21;
            x[17497098 + i] = (t144*t131 + t147*t132 + t150*t133)*x21;
            x[18495348 + i] = (t153*t131 + t156*t132 + t159*t133)*x21;
            x[19493598 + i] = (t131*t136 + t132*t139 + t142*t133)*x21;
            x[20491848 + i] = (t145*t131 + t148*t132 + t151*t133)*x21;
            x[21490098 + i] = (t154*t131 + t157*t132 + t160*t133)*x21;
            x[22488348 + i] = x21*((t131*t95 + t132*t96 + t133*t97)*t133 + ((t131*t75 + t132*t76 + t133*t77)*t131 + (t132*t86 + t131*t85 + t133*t87)*t132));
            x[23486598 + i] = x21*(t133*(t131*t98 + t132*t99 + t133*t100) + (t131*(t131*t78 + t132*t79 + t133*t80) + t132*(t131*t88 + t132*t89 + t133*t90)));
            x[24484848 + i] = ((x12*t72 + x13*t73 + x14*t74)*t131 + (x12*t82 + x13*t83 + x14*t84)*t132 + (x12*t92 + x13*t93 + x14*t94)*t133)*x21;
            x[25483098 + i] = (t131*t167 + t132*t170 + t173*t133)*x21;
            x[26481348 + i] = (t176*t131 + t179*t132 + t182*t133)*x21;
            x[27479598 + i] = (t161*t131 + t163*t132 + t165*t133)*x21;
            x[28477848 + i] = (t131*t168 + t132*t171 + t174*t133)*x21;
            x[29476098 + i] = (t177*t131 + t180*t132 + t183*t133)*x21;
            x[30474348 + i] = (t162*t131 + t164*t132 + t166*t133)*x21;
            x[31472598 + i] = (t131*t169 + t132*t172 + t175*t133)*x21;
            x[32470848 + i] = (t178*t131 + t181*t132 + t184*t133)*x21;
            x[33469098 + i] = x21*((t131*t128 + t132*t129 + t133*t130)*t133 + ((t131*t108 + t132*t109 + t133*t110)*t131 + (t132*t119 + t131*t118 + t133*t120)*t132));
            x[34467348 + i] = ((x12*t102 + x13*t103 + x14*t104)*t131 + (x12*t112 + x13*t113 + x14*t114)*t132 + (x12*t122 + x13*t123 + x14*t124)*t133)*x21;
            x[35465598 + i] = ((x12*t105 + x13*t106 + x14*t107)*t131 + (x12*t115 + x13*t116 + x14*t117)*t132 + (x12*t125 + x13*t126 + x14*t127)*t133)*x21;
            x[36463848 + i] = (t131*t197 + t132*t200 + t203*t133)*x21;
            x[37462098 + i] = (t185*t131 + t187*t132 + t189*t133)*x21;
            x[38460348 + i] = (t191*t131 + t193*t132 + t195*t133)*x21;
            x[39458598 + i] = (t131*t198 + t132*t201 + t204*t133)*x21;
            x[40456848 + i] = (t186*t131 + t188*t132 + t190*t133)*x21;
            x[41455098 + i] = (t192*t131 + t194*t132 + t196*t133)*x21;
            x[42453348 + i] = (t131*t199 + t132*t202 + t205*t133)*x21;
            x[43451598 + i] = x21*(x12*t134 + x13*t137 + x14*t140);
            x[44449848 + i] = (x14*t149 + (x12*t143 + x13*t146))*x21;
            x[45448098 + i] = (x14*t158 + (x12*t152 + x13*t155))*x21;
            x[46446348 + i] = x21*(x12*t135 + x13*t138 + x14*t141);
            x[47444598 + i] = (x14*t150 + (x12*t144 + x13*t147))*x21;
            x[48442848 + i] = (x14*t159 + (x12*t153 + x13*t156))*x21;
            x[49441098 + i] = x21*(x12*t136 + x13*t139 + x14*t142);
            x[50439348 + i] = (x14*t151 + (x12*t145 + x13*t148))*x21;
            x[51437598 + i] = (x14*t160 + (x12*t154 + x13*t157))*x21;
            x[52435848 + i] = x21*(x12*t167 + x13*t170 + x14*t173);
            x[53434098 + i] = (x14*t182 + (x12*t176 + x13*t179))*x21;
            x[54432348 + i] = (x14*t165 + (x12*t161 + x13*t163))*x21;
            x[55430598 + i] = x21*(x12*t168 + x13*t171 + x14*t174);
            x[56428848 + i] = (x14*t183 + (x12*t177 + x13*t180))*x21;
            x[57427098 + i] = (x14*t166 + (x12*t162 + x13*t164))*x21;
            x[58425348 + i] = x21*(x12*t169 + x13*t172 + x14*t175);
            x[59423598 + i] = (x14*t184 + (x12*t178 + x13*t181))*x21;
            x[60421848 + i] = x21*(x12*t197 + x13*t200 + x14*t203);
            x[61420098 + i] = (x14*t189 + (x12*t185 + x13*t187))*x21;
            x[62418348 + i] = (x14*t195 + (x12*t191 + x13*t193))*x21;
            x[63416598 + i] = x21*(x12*t198 + x13*t201 + x14*t204);
            x[64414848 + i] = (x14*t190 + (x12*t186 + x13*t188))*x21;
            x[65413098 + i] = (x14*t196 + (x12*t192 + x13*t194))*x21;
            x[66411348 + i] = x21*(x12*t199 + x13*t202 + x14*t205);
            x[67409598 + i] = x21*(x15*t135 + x16*t138 + x17*t141);
            x[68407848 + i] = (x17*t150 + (x15*t144 + x16*t147))*x21;
            x[69406098 + i] = (x17*t159 + (x15*t153 + x16*t156))*x21;
            x[70404348 + i] = x21*(x15*t136 + x16*t139 + x17*t142);
            x[71402598 + i] = (x17*t151 + (x15*t145 + x16*t148))*x21;
            x[72400848 + i] = (x17*t160 + (x15*t154 + x16*t157))*x21;
            x[73399098 + i] = x21*(x15*t168 + x16*t171 + x17*t174);
            x[74397348 + i] = (x17*t183 + (x15*t177 + x16*t180))*x21;
            x[75395598 + i] = (x17*t166 + (x15*t162 + x16*t164))*x21;
            x[76393848 + i] = x21*(x15*t169 + x16*t172 + x17*t175);
            x[77392098 + i] = (x17*t184 + (x15*t178 + x16*t181))*x21;
            x[78390348 + i] = x21*(x15*t198 + x16*t201 + x17*t204);
            x[79388598 + i] = (x17*t190 + (x15*t186 + x16*t188))*x21;
            x[80386848 + i] = (x17*t196 + (x15*t192 + x16*t194))*x21;
            x[81385098 + i] = x21*(x15*t199 + x16*t202 + x17*t205);
            x[82383348 + i] = x21*(x18*t136 + x19*t139 + x20*t142);
            x[83381598 + i] = (x20*t151 + (x18*t145 + x19*t148))*x21;
            x[84379848 + i] = (x20*t160 + (x18*t154 + x19*t157))*x21;
            x[85378098 + i] = x21*(x18*t169 + x19*t172 + x20*t175);
            x[86376348 + i] = (x20*t184 + (x18*t178 + x19*t181))*x21;
            x[87374598 + i] = x21*(x18*t199 + x19*t202 + x20*t205);
        }
    }
    for (long i = 998248; i < 998250; ++i) {
        const double x0 = x[p[0 + i]];
        const double x1 = x[p[0 + i] + 1];
        const double x2 = x[p[0 + i] + 2];
        const double x3 = x[p[998250 + i]];
        const double x4 = x[p[1996500 + i]];
        const double x5 = x[p[2994750 + i]];
        const double x6 = x[p[3993000 + i]];
        const double x7 = x[p[4991250 + i]];
        const double x8 = x[p[5989500 + i]];
        const double x9 = x[p[0 + i] + 9579];
        const double x10 = x[p[0 + i] + 9580];
        const double x11 = x[p[0 + i] + 9581];
        const double x12 = x[p[6987750 + i]];
        const double x13 = x[p[7986000 + i]];
        const double x14 = x[p[8984250 + i]];
        const double x15 = x[p[9982500 + i]];
        const double x16 = x[p[10980750 + i]];
        const double x17 = x[p[11979000 + i]];
        const double x18 = x[p[12977250 + i]];
        const double x19 = x[p[13975500 + i]];
        const double x20 = x[p[14973750 + i]];
        const double x21 = x[p[15972000 + i]];
        const double t0 = x3 - x0;
        const double t1 = x6 - x0;
        const double t2 = x9 - x0;
        const double t3 = x4 - x1;
        const double t4 = x7 - x1;
        const double t5 = x10 - x1;
        const double t6 = x5 - x2;
        const double t7 = x8 - x2;
        const double t8 = x11 - x2;
        const double t9 = x12*t0 + x15*t1 + x18*t2;
        const double t10 = x13*t0 + x16*t1 + x19*t2;
        const double t11 = x14*t0 + x17*t1 + x20*t2;
        const double t12 = x12*t3 + x15*t4 + x18*t5;
        const double t13 = x13*t3 + x16*t4 + x19*t5;
        const double t14 = x14*t3 + x17*t4 + x20*t5;
        const double t15 = x12*t6 + x15*t7 + x18*t8;
        const double t16 = x13*t6 + x16*t7 + x19*t8;
        const double t17 = x14*t6 + x17*t7 + x20*t8;
        const double t18 = t13*t17 - t14*t16;
        const double t19 = t14*t15 - t12*t17;
        const double t20 = t12*t16 - t13*t15;
        const double t21 = t18*t9 + t19*t10 + t20*t11;
        const double t22 = t18/t21;
        const double t23 = (t11*t16 - t10*t17)/t21;
        const double t24 = (t10*t14 - t11*t13)/t21;
        const double t25 = t19/t21;
        const double t26 = (t9*t17 - t11*t15)/t21;
        const double t27 = (t11*t12 - t9*t14)/t21;
        const double t28 = t20/t21;
        const double t29 = (t10*t15 - t9*t16)/t21;
        const double t30 = (t9*t13 - t10*t12)/t21;
        const double t31 = 1.0 - log(t21)*10.0;
        const double t32 = t22*t31;
        const double t33 = t22*10.0;
        const double t34 = t32*t22 + t33*t22 + 1.0;
        const double t35 = t32*t25 + t33*t25;
        const double t36 = t32*t28 + t33*t28;
        const double t37 = t23*t31;
        const double t38 = t37*t22 + t33*t23;
        const double t39 = t37*t25 + t33*t26;
        const double t40 = t37*t28 + t33*t29;
        const double t41 = t24*t31;
        const double t42 = t41*t22 + t33*t24;
        const double t43 = t41*t25 + t33*t27;
        const double t44 = t41*t28 + t33*t30;
        const double t45 = t25*t31;
        const double t46 = t25*10.0;
        const double t47 = t45*t22 + t46*t22;
        const double t48 = t45*t25 + t46*t25 + 1.0;
        const double t49 = t45*t28 + t46*t28;
        const double t50 = t26*t31;
        const double t51 = t50*t22 + t46*t23;
        const double t52 = t50*t25 + t46*t26;
        const double t53 = t50*t28 + t46*t29;
        const double t54 = t27*t31;
        const double t55 = t54*t22 + t46*t24;
        const double t56 = t54*t25 + t46*t27;
        const double t57 = t54*t28 + t46*t30;
        const double t58 = t28*t31;
        const double t59 = t28*10.0;
        const double t60 = t58*t22 + t59*t22;
        const double t61 = t58*t25 + t59*t25;
        const double t62 = t58*t28 + t59*t28 + 1.0;
        const double t63 = t29*t31;
        const double t64 = t63*t22 + t59*t23;
        const double t65 = t63*t25 + t59*t26;
        const double t66 = t63*t28 + t59*t29;
        const double t67 = t30*t31;
        const double t68 = t67*t22 + t59*t24;
        const double t69 = t67*t25 + t59*t27;
        const double t70 = t67*t28 + t59*t30;
        const double t71 = t23*10.0;
        const double t72 = t32*t23 + t71*t22;
        const double t73 = t32*t26 + t71*t25;
        const double t74 = t32*t29 + t71*t28;
        const double t75 = t37*t23 + t71*t23 + 1.0;
        const double t76 = t37*t26 + t71*t26;
        const double t77 = t37*t29 + t71*t29;
        const double t78 = t41*t23 + t71*t24;
        const double t79 = t41*t26 + t71*t27;
        const double t80 = t41*t29 + t71*t30;
        const double t81 = t26*10.0;
        const double t82 = t45*t23 + t81*t22;
        const double t83 = t45*t26 + t81*t25;
        const double t84 = t45*t29 + t81*t28;
        const double t85 = t50*t23 + t81*t23;
        const double t86 = t50*t26 + t81*t26 + 1.0;
        const double t87 = t50*t29 + t81*t29;
        const double t88 = t54*t23 + t81*t24;
        const double t89 = t54*t26 + t81*t27;
        const double t90 = t54*t29 + t81*t30;
        const double t91 = t29*10.0;
        const double t92 = t58*t23 + t91*t22;
        const double t93 = t58*t26 + t91*t25;
        const double t94 = t58*t29 + t91*t28;
        const double t95 = t63*t23 + t91*t23;
        const double t96 = t63*t26 + t91*t26;
        const double t97 = t63*t29 + t91*t29 + 1.0;
        const double t98 = t67*t23 + t91*t24;
        const double t99 = t67*t26 + t91*t27;
        const double t100 = t67*t29 + t91*t30;
        const double t101 = t24*10.0;
        const double t102 = t32*t24 + t101*t22;
        const double t103 = t32*t27 + t101*t25;
        const double t104 = t32*t30 + t101*t28;
        const double t105 = t37*t24 + t101*t23;
        const double t106 = t37*t27 + t101*t26;
        const double t107 = t37*t30 + t101*t29;
        const double t108 = t41*t24 + t101*t24 + 1.0;
        const double t109 = t41*t27 + t101*t27;
        const double t110 = t41*t30 + t101*t30;
        const double t111 = t27*10.0;
        const double t112 = t45*t24 + t111*t22;
        const double t113 = t45*t27 + t111*t25;
        const double t114 = t45*t30 + t111*t28;
        const double t115 = t50*t24 + t111*t23;
        const double t116 = t50*t27 + t111*t26;
        const double t117 = t50*t30 + t111*t29;
        const double t118 = t54*t24 + t111*t24;
        const double t119 = t54*t27 + t111*t27 + 1.0;
        const double t120 = t54*t30 + t111*t30;
        const double t121 = t30*10.0;
        const double t122 = t58*t24 + t121*t22;
        const double t123 = t58*t27 + t121*t25;
        const double t124 = t58*t30 + t121*t28;
        const double t125 = t63*t24 + t121*t23;
        const double t126 = t63*t27 + t121*t26;
        const double t127 = t63*t30 + t121*t29;
        const double t128 = t67*t24 + t121*t24;
        const double t129 = t67*t27 + t121*t27;
        const double t130 = t67*t30 + t121*t30 + 1.0;
        const double t131 = -(x18 + (x12 + x15));
        const double t132 = -(x19 + (x13 + x16));
        const double t133 = -(x20 + (x14 + x17));
        const double t134 = x13*t35 + x12*t34 + x14*t36;
        const double t135 = x16*t35 + x15*t34 + x17*t36;
        const double t136 = x19*t35 + x18*t34 + x20*t36;
        const double t137 = x12*t47 + x13*t48 + x14*t49;
        const double t138 = x15*t47 + x16*t48 + x17*t49;
        const double t139 = x18*t47 + x19*t48 + x20*t49;
        const double t140 = x12*t60 + x13*t61 + x14*t62;
        const double t141 = x15*t60 + x16*t61 + x17*t62;
        const double t142 = x18*t60 + x19*t61 + x20*t62;
        const double t143 = x12*t38 + x13*t39 + x14*t40;
        const double t144 = x15*t38 + x16*t39 + x17*t40;
        const double t145 = x18*t38 + x19*t39 + x20*t40;
        const double t146 = x12*t51 + x13*t52 + x14*t53;
        const double t147 = x15*t51 + x16*t52 + x17*t53;
        const double t148 = x18*t51 + x19*t52 + x20*t53;
        const double t149 = x12*t64 + x13*t65 + x14*t66;
        const double t150 = x15*t64 + x16*t65 + x17*t66;
        const double t151 = x18*t64 + x19*t65 + x20*t66;
        const double t152 = x12*t42 + x13*t43 + x14*t44;
        const double t153 = x15*t42 + x16*t43 + x17*t44;
        const double t154 = x18*t42 + x19*t43 + x20*t44;
        const double t155 = x12*t55 + x13*t56 + x14*t57;
        const double t156 = x15*t55 + x16*t56 + x17*t57;
        const double t157 = x18*t55 + x19*t56 + x20*t57;
        const double t158 = x12*t68 + x13*t69 + x14*t70;
        const double t159 = x15*t68 + x16*t69 + x17*t70;
        const double t160 = x18*t68 + x19*t69 + x20*t70;
        const double t161 = x15*t72 + x16*t73 + x17*t74;
        const double t162 = x18*t72 + x19*t73 + x20*t74;
        const double t163 = x15*t82 + x16*t83 + x17*t84;
        const double t164 = x18*t82 + x19*t83 + x20*t84;
        const double t165 = x15*t92 + x16*t93 + x17*t94;
        const double t166 = x18*t92 + x19*t93 + x20*t94;
        const double t167 = x13*t76 + x12*t75 + x14*t77;
        const double t168 = x16*t76 + x15*t75 + x17*t77;
        const double t169 = x19*t76 + x18*t75 + x20*t77;
        const double t170 = x12*t85 + x13*t86 + x14*t87;
        const double t171 = x15*t85 + x16*t86 + x17*t87;
        const double t172 = x18*t85 + x19*t86 + x20*t87;
        const double t173 = x12*t95 + x13*t96 + x14*t97;
        const double t174 = x15*t95 + x16*t96 + x17*t97;
        const double t175 = x18*t95 + x19*t96 + x20*t97;
        const double t176 = x12*t78 + x13*t79 + x14*t80;
        const double t177 = x15*t78 + x16*t79 + x17*t80;
        const double t178 = x18*t78 + x19*t79 + x20*t80;
        const double t179 = x12*t88 + x13*t89 + x14*t90;
        const double t180 = x15*t88 + x16*t89 + x17*t90;
        const double t181 = x18*t88 + x19*t89 + x20*t90;
        const double t182 = x12*t98 + x13*t99 + x14*t100;
        const double t183 = x15*t98 + x16*t99 + x17*t100;
        const double t184 = x18*t98 + x19*t99 + x20*t100;
        const double t185 = x15*t102 + x16*t103 + x17*t104;
        const double t186 = x18*t102 + x19*t103 + x20*t104;
        const double t187 = x15*t112 + x16*t113 + x17*t114;
        const double t188 = x18*t112 + x19*t113 + x20*t114;
        const double t189 = x15*t122 + x16*t123 + x17*t124;
        const double t190 = x18*t122 + x19*t123 + x20*t124;
        const double t191 = x15*t105 + x16*t106 + x17*t107;
        const double t192 = x18*t105 + x19*t106 + x20*t107;
        const double t193 = x15*t115 + x16*t116 + x17*t117;
        const double t194 = x18*t115 + x19*t116 + x20*t117;
        const double t195 = x15*t125 + x16*t126 + x17*t127;
        const double t196 = x18*t125 + x19*t126 + x20*t127;
        const double t197 = x13*t109 + x12*t108 + x14*t110;
        const double t198 = x16*t109 + x15*t108 + x17*t110;
        const double t199 = x19*t109 + x18*t108 + x20*t110;
        const double t200 = x12*t118 + x13*t119 + x14*t120;
        const double t201 = x15*t118 + x16*t119 + x17*t120;
        const double t202 = x18*t118 + x19*t119 + x20*t120;
        const double t203 = x12*t128 + x13*t129 + x14*t130;
        const double t204 = x15*t128 + x16*t129 + x17*t130;
        const double t205 = x18*t128 + x19*t129 + x20*t130;
        x[10509348 + i] = x21*((t131*t60 + t132*t61 + t133*t62)*t133 + ((t131*t34 + t132*t35 + t133*t36)*t131 + (t132*t48 + t131*t47 + t133*t49)*t132));
        x[11507598 + i] = x21*(t133*(t131*t64 + t132*t65 + t133*t66) + (t131*(t131*t38 + t132*t39 + t133*t40) + t132*(t131*t51 + t132*t52 + t133*t53)));
        x[12505848 + i] = x21*(t133*(t131*t68 + t132*t69 + t133*t70) + (t131*(t131*t42 + t132*t43 + t133*t44) + t132*(t131*t55 + t132*t56 + t133*t57)));
        x[13504098 + i] = (t131*t134 + t132*t137 + t140*t133)*x21;
        x[14502348 + i] = (t143*t131 + t146*t132 + t149*t133)*x21;
        x[15500598 + i] = (t152*t131 + t155*t132 + t158*t133)*x21;
        x[16498848 + i] = (t131*t135 + t132*t138 + t141*t133)*x21;
        x[17497098 + i] = (t144*t131 + t147*t132 + t150*t133)*x21;
        x[18495348 + i] = (t153*t131 + t156*t132 + t159*t133)*x21;
        x[19493598 + i] = (t131*t136 + t132*t139 + t142*t133)*x21;
        x[20491848 + i] = (t145*t131 + t148*t132 + t151*t133)*x21;
        x[21490098 + i] = (t154*t131 + t157*t132 + t160*t133)*x21;
        x[22488348 + i] = x21*((t131*t95 + t132*t96 + t133*t97)*t133 + ((t131*t75 + t132*t76 + t133*t77)*t131 + (t132*t86 + t131*t85 + t133*t87)*t132));
        x[23486598 + i] = x21*(t133*(t131*t98 + t132*t99 + t133*t100) + (t131*(t131*t78 + t132*t79 + t133*t80) + t132*(t131*t88 + t132*t89 + t133*t90)));
        x[24484848 + i] = ((x12*t72 + x13*t73 + x14*t74)*t131 + (x12*t82 + x13*t83 + x14*t84)*t132 + (x12*t92 + x13*t93 + x14*t94)*t133)*x21;
        x[25483098 + i] = (t131*t167 + t132*t170 + t173*t133)*x21;
        x[26481348 + i] = (t176*t131 + t179*t132 + t182*t133)*x21;
        x[27479598 + i] = (t161*t131 + t163*t132 + t165*t133)*x21;
        x[28477848 + i] = (t131*t168 + t132*t171 + t174*t133)*x21;
        x[29476098 + i] = (t177*t131 + t180*t132 + t183*t133)*x21;
        x[30474348 + i] = (t162*t131 + t164*t132 + t166*t133)*x21;
        x[31472598 + i] = (t131*t169 + t132*t172 + t175*t133)*x21;
        x[32470848 + i] = (t178*t131 + t181*t132 + t184*t133)*x21;
        x[33469098 + i] = x21*((t131*t128 + t132*t129 + t133*t130)*t133 + ((t131*t108 + t132*t109 + t133*t110)*t131 + (t132*t119 + t131*t118 + t133*t120)*t132));
        x[34467348 + i] = ((x12*t102 + x13*t103 + x14*t104)*t131 + (x12*t112 + x13*t113 + x14*t114)*t132 + (x12*t122 + x13*t123 + x14*t124)*t133)*x21;
        x[35465598 + i] = ((x12*t105 + x13*t106 + x14*t107)*t131 + (x12*t115 + x13*t116 + x14*t117)*t132 + (x12*t125 + x13*t126 + x14*t127)*t133)*x21;
        x[36463848 + i] = (t131*t197 + t132*t200 + t203*t133)*x21;
        x[37462098 + i] = (t185*t131 + t187*t132 + t189*t133)*x21;
        x[38460348 + i] = (t191*t131 + t193*t132 + t195*t133)*x21;
        x[39458598 + i] = (t131*t198 + t132*t201 + t204*t133)*x21;
        x[40456848 + i] = (t186*t131 + t188*t132 + t190*t133)*x21;
        x[41455098 + i] = (t192*t131 + t194*t132 + t196*t133)*x21;
        x[42453348 + i] = (t131*t199 + t132*t202 + t205*t133)*x21;
        x[43451598 + i] = x21*(x12*t134 + x13*t137 + x14*t140);
        x[44449848 + i] = (x14*t149 + (x12*t143 + x13*t146))*x21;
        x[45448098 + i] = (x14*t158 + (x12*t152 + x13*t155))*x21;
        x[46446348 + i] = x21*(x12*t135 + x13*t138 + x14*t141);
        x[47444598 + i] = (x14*t150 + (x12*t144 + x13*t147))*x21;
        x[48442848 + i] = (x14*t159 + (x12*t153 + x13*t156))*x21;
        x[49441098 + i] = x21*(x12*t136 + x13*t139 + x14*t142);
        x[50439348 + i] = (x14*t151 + (x12*t145 + x13*t148))*x21;
        x[51437598 + i] = (x14*t160 + (x12*t154 + x13*t157))*x21;
        x[52435848 + i] = x21*(x12*t167 + x13*t170 + x14*t173);
        x[53434098 + i] = (x14*t182 + (x12*t176 + x13*t179))*x21;
        x[54432348 + i] = (x14*t165 + (x12*t161 + x13*t163))*x21;
        x[55430598 + i] = x21*(x12*t168 + x13*t171 + x14*t174);
        x[56428848 + i] = (x14*t183 + (x12*t177 + x13*t180))*x21;
        x[57427098 + i] = (x14*t166 + (x12*t162 + x13*t164))*x21;
        x[58425348 + i] = x21*(x12*t169 + x13*t172 + x14*t175);
        x[59423598 + i] = (x14*t184 + (x12*t178 + x13*t181))*x21;
        x[60421848 + i] = x21*(x12*t197 + x13*t200 + x14*t203);
        x[61420098 + i] = (x14*t189 + (x12*t185 + x13*t187))*x21;
        x[62418348 + i] = (x14*t195 + (x12*t191 + x13*t193))*x21;
        x[63416598 + i] = x21*(x12*t198 + x13*t201 + x14*t204);
        x[64414848 + i] = (x14*t190 + (x12*t186 + x13*t188))*x21;
        x[65413098 + i] = (x14*t196 + (x12*t192 + x13*t194))*x21;
        x[66411348 + i] = x21*(x12*t199 + x13*t202 + x14*t205);
        x[67409598 + i] = x21*(x15*t135 + x16*t138 + x17*t141);
        x[68407848 + i] = (x17*t150 + (x15*t144 + x16*t147))*x21;
        x[69406098 + i] = (x17*t159 + (x15*t153 + x16*t156))*x21;
        x[70404348 + i] = x21*(x15*t136 + x16*t139 + x17*t142);
        x[71402598 + i] = (x17*t151 + (x15*t145 + x16*t148))*x21;
        x[72400848 + i] = (x17*t160 + (x15*t154 + x16*t157))*x21;
        x[73399098 + i] = x21*(x15*t168 + x16*t171 + x17*t174);
        x[74397348 + i] = (x17*t183 + (x15*t177 + x16*t180))*x21;
        x[75395598 + i] = (x17*t166 + (x15*t162 + x16*t164))*x21;
        x[76393848 + i] = x21*(x15*t169 + x16*t172 + x17*t175);
        x[77392098 + i] = (x17*t184 + (x15*t178 + x16*t181))*x21;
        x[78390348 + i] = x21*(x15*t198 + x16*t201 + x17*t204);
        x[79388598 + i] = (x17*t190 + (x15*t186 + x16*t188))*x21;
        x[80386848 + i] = (x17*t196 + (x15*t192 + x16*t194))*x21;
        x[81385098 + i] = x21*(x15*t199 + x16*t202 + x17*t205);
        x[82383348 + i] = x21*(x18*t136 + x19*t139 + x20*t142);
        x[83381598 + i] = (x20*t151 + (x18*t145 + x19*t148))*x21;
        x[84379848 + i] = (x20*t160 + (x18*t154 + x19*t157))*x21;
        x[85378098 + i] = x21*(x18*t169 + x19*t172 + x20*t175);
        x[86376348 + i] = (x20*t184 + (x18*t178 + x19*t181))*x21;
        x[87374598 + i] = x21*(x18*t199 + x19*t202 + x20*t205);
    }
}

/* level 1, 166356 instance(s), 1 result(s) each */
static void nh_sum2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 41589; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[16970250 + i]];
            const double x1 = x[p[17136606 + i]];
            x[88372848 + i] = x0 + x1;
        }
    }
}

/* level 1, 320760 instance(s), 1 result(s) each */
static void nh_sum3(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 80190; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[17302962 + i]];
            const double x1 = x[p[17623722 + i]];
            const double x2 = x[p[17944482 + i]];
            x[88539204 + i] = x0 + x1 + x2;
        }
    }
}

/* level 1, 4412394 instance(s), 1 result(s) each */
static void nh_sum4(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 1103098; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[18265242 + i]];
            const double x1 = x[p[22677636 + i]];
            const double x2 = x[p[27090030 + i]];
            const double x3 = x[p[31502424 + i]];
            x[88859964 + i] = x0 + x1 + x2 + x3;
        }
    }
    for (long i = 4412392; i < 4412394; ++i) {
        const double x0 = x[p[18265242 + i]];
        const double x1 = x[p[22677636 + i]];
        const double x2 = x[p[27090030 + i]];
        const double x3 = x[p[31502424 + i]];
        x[88859964 + i] = x0 + x1 + x2 + x3;
    }
}

/* level 1, 5827647 instance(s), 1 result(s) each */
static void nh_sum6(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 1456911; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[35914818 + i]];
            const double x1 = x[p[41742465 + i]];
            const double x2 = x[p[47570112 + i]];
            const double x3 = x[p[53397759 + i]];
            const double x4 = x[p[59225406 + i]];
            const double x5 = x[p[65053053 + i]];
            x[93272360 + i] = x0 + x1 + x2 + x3 + x4 + x5;
        }
    }
    for (long i = 5827644; i < 5827647; ++i) {
        const double x0 = x[p[35914818 + i]];
        const double x1 = x[p[41742465 + i]];
        const double x2 = x[p[47570112 + i]];
        const double x3 = x[p[53397759 + i]];
        const double x4 = x[p[59225406 + i]];
        const double x5 = x[p[65053053 + i]];
        x[93272360 + i] = x0 + x1 + x2 + x3 + x4 + x5;
    }
}

/* level 1, 1944 instance(s), 1 result(s) each */
static void nh_sum8(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 486; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[70880700 + i]];
            const double x1 = x[p[70880700 + i] + 1];
            const double x2 = x[p[70880700 + i] + 2];
            const double x3 = x[p[70880700 + i] + 3];
            const double x4 = x[p[70880700 + i] + 4];
            const double x5 = x[p[70880700 + i] + 5];
            const double x6 = x[p[70882644 + i]];
            const double x7 = x[p[70884588 + i]];
            x[99100008 + i] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
        }
    }
}

/* level 1, 104976 instance(s), 1 result(s) each */
static void nh_sum12(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 26244; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[70886532 + i]];
            const double x1 = x[p[70886532 + i] + 1];
            const double x2 = x[p[70886532 + i] + 2];
            const double x3 = x[p[70886532 + i] + 3];
            const double x4 = x[p[70886532 + i] + 4];
            const double x5 = x[p[70886532 + i] + 5];
            const double x6 = x[p[70991508 + i]];
            const double x7 = x[p[71096484 + i]];
            const double x8 = x[p[71201460 + i]];
            const double x9 = x[p[71306436 + i]];
            const double x10 = x[p[71411412 + i]];
            const double x11 = x[p[71516388 + i]];
            x[99101952 + i] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + x8 + x9 + x10 + x11;
        }
    }
}

/* level 1, 944784 instance(s), 1 result(s) each */
static void nh_sum24(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 236196; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[71621364 + i]];
            const double x1 = x[p[71621364 + i] + 1];
            const double x2 = x[p[71621364 + i] + 2];
            const double x3 = x[p[71621364 + i] + 3];
            const double x4 = x[p[71621364 + i] + 4];
            const double x5 = x[p[71621364 + i] + 5];
            const double x6 = x[p[72566148 + i]];
            const double x7 = x[p[73510932 + i]];
            const double x8 = x[p[74455716 + i]];
            const double x9 = x[p[75400500 + i]];
            const double x10 = x[p[76345284 + i]];
            const double x11 = x[p[77290068 + i]];
            const double x12 = x[p[78234852 + i]];
            const double x13 = x[p[79179636 + i]];
            const double x14 = x[p[80124420 + i]];
            const double x15 = x[p[81069204 + i]];
            const double x16 = x[p[82013988 + i]];
            const double x17 = x[p[82958772 + i]];
            const double x18 = x[p[83903556 + i]];
            const double x19 = x[p[84848340 + i]];
            const double x20 = x[p[85793124 + i]];
            const double x21 = x[p[86737908 + i]];
            const double x22 = x[p[87682692 + i]];
            const double x23 = x[p[88627476 + i]];
            x[99206928 + i] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + x8 + x9 + x10 + x11 + x12 + x13 + x14 + x15 + x16 + x17 + x18 + x19 + x20 + x21 + x22 + x23;
        }
    }
}

void sg_run(double* x, const double* c, const unsigned* p) {
    nh_elem(x, c, p);
    nh_sum2(x, c, p);
    nh_sum3(x, c, p);
    nh_sum4(x, c, p);
    nh_sum6(x, c, p);
    nh_sum8(x, c, p);
    nh_sum12(x, c, p);
    nh_sum24(x, c, p);
}
